// prep.cu -- per-polygon prep.
//
// For each ring: the half-open pixel MBR; the area by the shoelace formula
// A = 1/2 |sum_i (x_i y_{i+1} - x_{i+1} y_i)| with "different threads compute
// different vertices and sum up the partial results" (§3.2),
// evaluated on MBR-rebased coordinates in int64 (translation invariant, no
// overflow); validation (rectilinear edges, ranges, offsets); the 8-byte edge
// records PixelBox streams (vertical edges compacted to the front of the
// polygon's vertex slot, horizontal edges to the back); and the per-set
// statistics the grid-hash join sizes its grid from.
//
// A CTA stages the vertex range of 128 consecutive polygons in shared memory
// with one TMA bulk copy, derives each small polygon by one thread (large ones
// by a warp) in place, and writes the slots back with one TMA bulk store.
// Ranges larger than the tile fall back to reading the polygon's vertices from
// global memory (warp per polygon).
#include "packed_decode.cuh"

namespace sccg {

#ifndef SCCG_PREP_THREADS
#define SCCG_PREP_THREADS 128
#endif
#ifndef SCCG_PREP_VERTS
#define SCCG_PREP_VERTS 5120
#endif
constexpr int kPrepThreads = SCCG_PREP_THREADS;
constexpr int kPrepPolys = kPrepThreads;  // one ring per thread per tile
static_assert(kPrepThreads % 32 == 0 && kPrepThreads <= 256, "whole warps; ring indices fit a byte");
constexpr int kPrepVerts = SCCG_PREP_VERTS;
#ifndef SCCG_PREP_RES_DEAL
#define SCCG_PREP_RES_DEAL 2  // 0: V-sorted order, 1: residue-sorted alternation, 2: residue occurrences alternated
#endif
#ifndef SCCG_PREP_USED_ONLY
#define SCCG_PREP_USED_ONLY 0  // 1: write back only each ring's defined words, one bulk store per ring (measured slower: 177 vs 168 us on C2)
#endif
#ifndef SCCG_PREP_L2_PREFETCH
#define SCCG_PREP_L2_PREFETCH 2  // 0: off, 1: after the ring phase, 2: before it (measured best)
#endif
constexpr size_t kPrepSmem = kPrepVerts * sizeof(int2);  // 40 KB of int2 staged per tile (dynamic shared memory)


// ---- 1-D bulk copies on the TMA engine (cp.async.bulk): the tile is staged
// and written back without LSU traffic.  Addresses 16-byte aligned, sizes a
// multiple of 16.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
// SCCG_PREP_EVICT_FIRST: the vertex tiles are read once per step (nothing
// downstream of prep on the nucleus path reads xy), so their L2 lines are
// marked evict-first and the derived buffers PixelBox reads next keep L2.
#ifndef SCCG_PREP_RASTER
#define SCCG_PREP_RASTER 1  // memoized pixelization: prep stores each eligible ring's raster rows
#endif
#ifndef SCCG_PREP_EVICT_FIRST
#define SCCG_PREP_EVICT_FIRST 0
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
#if SCCG_PREP_EVICT_FIRST
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy_evict_first())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
#endif
}
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
#if SCCG_PREP_EVICT_FIRST
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;\n" ::"l"(src), "r"(bytes),
               "l"(policy_evict_first())
               : "memory");
#else
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra.uni WAIT%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_store_drain() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Predicated shared-memory store / return-free XOR reduction (no divergent
// branch around a conditional access).
__device__ __forceinline__ void sts64_if(unsigned saddr, unsigned lo, unsigned hi, bool c) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.shared.v2.u32 [%0], {%1, %2};\n}\n" ::"r"(saddr),
               "r"(lo), "r"(hi), "r"((unsigned)c)
               : "memory");
}
__device__ __forceinline__ void red_xor_if(unsigned saddr, unsigned v, bool c) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.shared.xor.b32 [%0], %1;\n}\n" ::"r"(saddr),
               "r"(v), "r"((unsigned)c)
               : "memory");
}

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bit, int64_t poly) {
  atomicOr(&status[0], bit);
  atomicMin(&status[1], (uint32_t)min(poly, (int64_t)0x7fffffff));
}

// One polygon by one warp.  `v` points at its first vertex (shared or
// global); vertical-edge records are written to `out` (compacted, ring order).
// When out aliases v (shared-memory tile) the writes are safe: a record lands
// at or before the vertex slot the warp has already read in this chunk.
__device__ __forceinline__ int4 prep_polygon(const int2* v, int64_t V, int64_t poly, uint64_t* out,
                                             int4* __restrict__ mbr, int64_t* __restrict__ area,
                                             int2* __restrict__ ecount, uint32_t* __restrict__ status,
                                             int validate, bool rast_ok, int& nv_out) {
  nv_out = 0;
  const int lane = threadIdx.x & 31;
  int xmin = INT_MAX, ymin = INT_MAX, xmax = INT_MIN, ymax = INT_MIN;
  for (int64_t i = lane; i < V; i += 32) {
    const int2 a = v[i];
    xmin = min(xmin, a.x);
    xmax = max(xmax, a.x);
    ymin = min(ymin, a.y);
    ymax = max(ymax, a.y);
  }
  xmin = __reduce_min_sync(0xffffffffu, xmin);
  ymin = __reduce_min_sync(0xffffffffu, ymin);
  xmax = __reduce_max_sync(0xffffffffu, xmax);
  ymax = __reduce_max_sync(0xffffffffu, ymax);
  const int4 m = make_int4(xmin, ymin, xmax, ymax);
  const bool bad_range = (int64_t)xmin < -kMaxCoord || (int64_t)xmax > kMaxCoord || (int64_t)ymin < -kMaxCoord ||
                         (int64_t)ymax > kMaxCoord || (int64_t)xmax - xmin > kMaxExtent ||
                         (int64_t)ymax - ymin > kMaxExtent;
  if (bad_range) {
    if (lane == 0) {
      mbr[poly] = m;
      area[poly] = 0;
      ecount[poly] = make_int2(0, 0);
      flag(status, SCCG_STATUS_RANGE, poly);
    }
    return m;
  }
  const int2 first = v[0];
  long long twice_area = 0;
  bool diag = false;
  int nvert = 0, nhor = 0;
  for (int64_t i0 = 0; i0 < V; i0 += 32) {
    const int64_t i = i0 + lane;
    bool is_v = false, is_h = false;
    uint64_t rec = 0;
    if (i < V) {
      const int2 a = v[i];
      const int2 c = i + 1 == V ? first : v[i + 1];
      const unsigned ax = a.x - xmin, ay = a.y - ymin, cx = c.x - xmin, cy = c.y - ymin;
      twice_area += (long long)(ax * cy) - (long long)(cx * ay);  // P:193, one term per thread
      is_v = ax == cx && ay != cy;
      is_h = ay == cy && ax != cx;
      diag |= ax != cx && ay != cy;
      rec = pack_edge(ax, min(ay, cy), max(ay, cy));
    }
    const unsigned bv = __ballot_sync(0xffffffffu, is_v);  // all lanes have read before anyone writes
    nhor += __popc(__ballot_sync(0xffffffffu, is_h));
    if (is_v) out[nvert + __popc(bv & lanemask_lt())] = rec;
    nvert += __popc(bv);
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) twice_area += __shfl_xor_sync(0xffffffffu, twice_area, o);
  diag = __any_sync(0xffffffffu, diag);
  nv_out = nvert;  // warp-uniform
  // Raster (as the thread path; ring in the shared-memory tile): lane per row,
  // each row word the XOR of the suffix masks of the records crossing it
  // (records read by broadcast), stored after the records.
  const int W = xmax - xmin, H = ymax - ymin;
  const bool raster = SCCG_PREP_RASTER && rast_ok && !diag && W <= 32 && H <= 128 && 2 * (V - nvert) >= H;
  if (raster) {
    unsigned* D = reinterpret_cast<unsigned*>(out + nvert);
    const unsigned wm = low_bits(W);
    for (int r0 = 0; r0 < H; r0 += 32) {
      const int r = r0 + lane;
      unsigned w = 0u;
      for (int k = 0; k < nvert; k++) {
        int c, lo, hi;
        unpack_edge(out[k], c, lo, hi);
        if (lo <= r && r < hi) w ^= shl_clamp(0xffffffffu, (unsigned)c);
      }
      if (r < H) D[r] = w & wm;
    }
    __syncwarp();
  }
  if (lane == 0) {
    area[poly] = (twice_area < 0 ? -twice_area : twice_area) / 2;
    mbr[poly] = m;
    ecount[poly] = make_int2(nvert | (raster ? kRasterFlag : 0), 0);  // records relative to the MBR origin: zero rebase
    (void)nhor;
    if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
  }
  return m;
}

// One polygon by one thread (the common small ring): same results as
// prep_polygon in ONE pass over the ring's vertices in the shared-memory tile
// (no separate MBR pass: shared-memory wavefronts bound this kernel).  The
// MBR is tracked on coordinates biased by 2^30 as unsigned (an out-of-range
// vertex shows up as a huge value, so the range check needs no extra test),
// and the records are written relative to the ring's FIRST vertex (16-bit
// fields mod 2^16); ecount[i].y = (x0 - xlo) | (y0 - ylo) << 16 rebases them
// to the MBR (decode_edge in internal.cuh).  Records are written in place
// over the ring's own vertex slot: record k lands in slot k <= i - 1 while
// vertex i is being read.
__device__ __forceinline__ int4 prep_polygon_thread(int2* v, int V, int rot, int64_t poly, int4* __restrict__ mbr,
                                                    int64_t* __restrict__ area, int2* __restrict__ ecount,
                                                    uint32_t* __restrict__ status, int validate, int& used8) {
  used8 = 0;
  constexpr unsigned kBias = 1u << 30;
  uint64_t* out = reinterpret_cast<uint64_t*>(v);
  const int2 f = v[0];
  const unsigned ux0 = (unsigned)f.x + kBias, uy0 = (unsigned)f.y + kBias;
  unsigned uxmin = ux0, uxmax = ux0, uymin = uy0, uymax = uy0;
  // Area: the shoelace of P:193 in trapezoid form, A = 1/2 |sum (x_i +
  // x_{i+1}) (y_{i+1} - y_i)| (the same sum re-associated), which on a
  // rectilinear ring is |sum over vertical edges of x_i (y_{i+1} - y_i)|
  // (horizontal edges add 0, vertical ones have x_i = x_{i+1}); on
  // coordinates relative to the first vertex (translation invariant: the
  // y-steps of a closed ring sum to 0), accumulated mod 2^32: exact whenever
  // A < 2^31, i.e. whenever W * H < 2^31 (else recomputed in int64 from the
  // records below).
  unsigned area32 = 0u;
  // edge classes by counts: nsx = edges with dx == 0, nsy = with dy == 0;
  // vertical = dx == 0 != dy (nvert), zero-length = nsx - nvert, horizontal =
  // nsy - (nsx - nvert), diagonal = V - nsy - nvert
  int nvert = 0, nsx = 0, nsy = 0;
  const unsigned sbase = smem_u32(out);
  int ax = 0, ay = 0;  // current vertex relative to the first
  auto edge = [&](int cx, int cy) {
    area32 += (unsigned)ax * (unsigned)(cy - ay);
    const bool same_x = ax == cx, same_y = ay == cy;
    const bool is_v = same_x && !same_y;
    nsx += same_x ? 1 : 0;
    nsy += same_y ? 1 : 0;
    // record: x | lo << 16 | hi << 32 | exit row << 48 (16-bit fields relative
    // to the first vertex; the exit row -- where the ring leaves the edge -- is
    // read by the raster pass below; decoders mask it off)
    const unsigned lo32 = __byte_perm(ax, min(ay, cy), 0x5410), hi32 = __byte_perm(max(ay, cy), cy, 0x5410);
    sts64_if(sbase + 8u * (unsigned)nvert, lo32, hi32, is_v);  // predicated: no divergent branch
    nvert += is_v ? 1 : 0;
    ax = cx;
    ay = cy;
  };
  auto vert = [&](const int2 c) {  // bias, MBR, relative coordinates
    const unsigned ux = (unsigned)c.x + kBias, uy = (unsigned)c.y + kBias;
    uxmin = min(uxmin, ux);
    uxmax = max(uxmax, ux);
    uymin = min(uymin, uy);
    uymax = max(uymax, uy);
    edge((int)(ux - ux0), (int)(uy - uy0));
  };
  // Vertices are loaded four at a time ahead of the record stores: the store of
  // edge i lands in slot <= i - 1, below every prefetched vertex, so loading
  // early is safe (the compiler cannot prove it and would otherwise serialise
  // each load behind the previous store).
  // 16-byte loads (two vertices each: a warp's lockstep loads then spread
  // over 8 bank quads instead of 16 bank pairs, fewer wavefronts per vertex)
  // after peeling one vertex when v + 1 is not 16-byte aligned
  int i = 1;
  if (V > 1 && (smem_u32(v + 1) & 15u) != 0u) {
    vert(v[1]);
    i = 2;
  }
  for (; i + 4 <= V; i += 4) {
    const int4 a = *reinterpret_cast<const int4*>(v + i), b = *reinterpret_cast<const int4*>(v + i + 2);
    vert(make_int2(a.x, a.y));
    vert(make_int2(a.z, a.w));
    vert(make_int2(b.x, b.y));
    vert(make_int2(b.z, b.w));
  }
  for (; i < V; i++) vert(v[i]);
  edge(0, 0);  // closing edge back to the first vertex
  const int4 m = make_int4((int)(uxmin - kBias), (int)(uymin - kBias), (int)(uxmax - kBias), (int)(uymax - kBias));
  mbr[poly] = m;
  // |coordinates| <= 2^30 <=> every biased value <= 2^31 (below -2^30 wraps to >= 2^32 - 2^30)
  if (uxmax > 2 * kBias || uymax > 2 * kBias || uxmax - uxmin > (unsigned)kMaxExtent ||
      uymax - uymin > (unsigned)kMaxExtent) {
    area[poly] = 0;
    ecount[poly] = make_int2(0, 0);
    flag(status, SCCG_STATUS_RANGE, poly);
    return m;
  }
  const unsigned ox = ux0 - uxmin, oy = uy0 - uymin;  // first vertex - MBR origin: rebases the records
  const int nhor = nsy - (nsx - nvert);
  (void)nhor;
  const bool diag = V - nsy - nvert != 0;
  const int W = (int)(uxmax - uxmin), H = (int)(uymax - uymin);
  if ((unsigned long long)W * (unsigned long long)H < (1ull << 31)) {
    const int a = (int)area32;
    area[poly] = a < 0 ? -a : a;
  } else {  // rare (a huge box): the same sum in int64 over the vertical records
    long long a = 0;
    for (int k = 0; k < nvert; k++) {
      const uint64_t r = out[k];
      int x, lo, hi;
      decode_edge(r, ox | (oy << 16), x, lo, hi);
      a += ((r >> 48) == ((r >> 32) & 0xffffu)) ? (long long)x * (hi - lo) : -(long long)x * (hi - lo);
    }
    area[poly] = a < 0 ? -a : a;
  }
  // Raster: pixel (x, y) of the MBR is inside
  // iff an odd number of the row's vertical edges lie at or left of x (R19) --
  // PIXELINPOLY depends on the polygon alone, so it is computed once here.
  // Row r as a 32-bit word (bit x = column xlo + x): difference trick -- each
  // vertical edge XORs its suffix mask into rows lo and hi (paired per row
  // below) -- then a prefix XOR over rows.  Stored in the slot's free tail (words 2 nv .. 2 nv + H), which
  // exists when 2 (V - nv) >= H; MBR width <= 32.
  bool raster = SCCG_PREP_RASTER && !diag && W <= 32 && 2 * (V - nvert) >= H;
  if (raster) {
    // In ring order a record's exit row is the next record's entry row -- y
    // only changes along vertical edges -- so every endpoint row gets both of
    // its suffix masks in ONE update: D[exit_k] ^= mask_k ^ mask_{k+1}
    // (cyclically).  Updates are predicated return-free shared reductions (no
    // branch, no load -> store chain), records read four at a time; the prefix
    // pass reads four rows ahead of its stores.
    unsigned* D = reinterpret_cast<unsigned*>(out + nvert);
    const unsigned dbase = sbase + 8u * (unsigned)nvert;
    // 8-byte accesses to D (it starts on an 8-byte boundary; an odd H leaves
    // one spare word in the slot, 2 (V - nv) >= H + 1): half the shared-memory
    // instructions of 4-byte ones
    uint2* D2 = reinterpret_cast<uint2*>(D);
    for (int r = 0; r < H; r += 2) D2[r >> 1] = make_uint2(0u, 0u);
    // The chain is cyclic and XOR is order-free, so each thread walks its
    // records from record s (the caller's rotation: the lockstep reads of a
    // warp's threads then hit distinct bank pairs, as far as the rings allow)
    // around to s - 1.
    const int s0 = nvert > 0 ? rot % nvert : 0;
    const uint64_t first = out[s0];
    unsigned mc = shl_clamp(0xffffffffu, ((unsigned)first + ox) & 0xffffu), yc = ((unsigned)(first >> 48) + oy) & 0xffffu;
    const unsigned m0 = mc;
    auto apply = [&](uint64_t nxt) {
      const unsigned mn = shl_clamp(0xffffffffu, ((unsigned)nxt + ox) & 0xffffu);
      red_xor_if(dbase + 4u * yc, mc ^ mn, yc < (unsigned)H);
      mc = mn;
      yc = ((unsigned)(nxt >> 48) + oy) & 0xffffu;
    };
    auto at = [&](int j) {  // record s0 + j, cyclically (j < nvert)
      const int k = s0 + j;
      return k < nvert ? k : k - nvert;
    };
    int j = 1;
    for (; j + 4 <= nvert; j += 4) {
      const uint64_t r0 = out[at(j)], r1 = out[at(j + 1)], r2 = out[at(j + 2)], r3 = out[at(j + 3)];
      apply(r0);
      apply(r1);
      apply(r2);
      apply(r3);
    }
    for (; j < nvert; j++) apply(out[at(j)]);
    red_xor_if(dbase + 4u * yc, mc ^ m0, yc < (unsigned)H);  // the last record's exit is the first record's entry
    unsigned acc = 0u;
    const unsigned wmask = low_bits(W);
    int r = 0;
    for (; r + 4 <= H; r += 4) {  // rows four ahead of their stores, two per access
      uint2 a = D2[r >> 1], b = D2[(r >> 1) + 1];
      acc ^= a.x;
      a.x = acc & wmask;
      acc ^= a.y;
      a.y = acc & wmask;
      acc ^= b.x;
      b.x = acc & wmask;
      acc ^= b.y;
      b.y = acc & wmask;
      D2[r >> 1] = a;
      D2[(r >> 1) + 1] = b;
    }
    for (; r < H; r += 2) {  // (an odd H also rewrites the spare word: not part of the raster)
      uint2 a = D2[r >> 1];
      acc ^= a.x;
      a.x = acc & wmask;
      acc ^= a.y;
      a.y = acc & wmask;
      D2[r >> 1] = a;
    }
  }
  ecount[poly] = make_int2(nvert | (raster ? kRasterFlag : 0), (int)(ox | (oy << 16)));
  if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
  used8 = nvert + (raster ? (H + 1) / 2 : 0);  // the slot's defined 8-byte words: records, then raster rows
  return m;
}

// Write back the defined part of one ring's slot -- its records (and raster
// rows) -- from the tile: the 16-byte-aligned body by one TMA bulk store, an
// odd first / last 8-byte word by plain stores.  The rest of the slot is left
// unwritten (nothing reads it), so the write traffic is what prep defines,
// not the whole vertex range.
__device__ __forceinline__ void store_used(uint64_t* __restrict__ edges, int64_t b, const uint64_t* src, int u) {
  if (u <= 0) return;
  const int64_t a0 = (b + 1) & ~int64_t(1), a1 = (b + u) & ~int64_t(1);
  fence_async_smem();  // this thread's shared-memory writes -> async proxy
  if (a1 > a0) bulk_store(edges + a0, src + (a0 - b), (unsigned)(a1 - a0) * 8u);
  if (b < a0) edges[b] = src[0];
  if (a1 < b + u && a1 >= a0) edges[a1] = src[a1 - b];
}

struct StatAcc {
  unsigned long long nonempty, sw, sh, swh;
  int bx0, by0, bx1, by1, mw, mh;
  __device__ __forceinline__ void init() {
    nonempty = sw = sh = swh = 0;
    bx0 = by0 = INT_MAX;
    bx1 = by1 = INT_MIN;
    mw = mh = 0;
  }
  __device__ __forceinline__ void add(const int4& m) {
    if (!(m.x < m.z && m.y < m.w)) return;
    const unsigned w1 = (unsigned)(m.z - m.x - 1), h1 = (unsigned)(m.w - m.y - 1);
    nonempty++;
    sw += w1;
    sh += h1;
    swh += (unsigned long long)w1 * h1;
    bx0 = min(bx0, m.x);
    by0 = min(by0, m.y);
    bx1 = max(bx1, m.z);
    by1 = max(by1, m.w);
    mw = max(mw, m.z - m.x);
    mh = max(mh, m.w - m.y);
  }
};

#ifndef SCCG_PREP_THREAD_MAXV
#define SCCG_PREP_THREAD_MAXV 192
#endif
constexpr int kThreadMaxV = SCCG_PREP_THREAD_MAXV;  // rings up to this size are prepped by one thread
#ifndef SCCG_PREP_SORT_SHIFT
#define SCCG_PREP_SORT_SHIFT 2  // counting-sort key = V >> shift
#endif
constexpr int kSortKeys = 64;     // counting-sort buckets (V / 4) for dealing rings to threads

// One launch preps up to kPrepMaxSets sets: their tiles form one index
// space, handed out by a device ticket (dynamic, so the last wave is short);
// a CTA flushes its statistics whenever it moves on to the next set.
constexpr int kPrepMaxSets = 4;
struct PrepSet {
  const int2* xy;
  const int64_t* off;
  int64_t n, nv_total;
  int4* mbr;
  int64_t* area;
  int2* ecount;
  uint64_t* edges;
  uint32_t* status;
  SetStats* stats;
  int bulk;
  // packed mode (sccg_prep_sets_packed): the rings come in the packed
  // transfer encoding; prep decodes each tile into shared memory and writes
  // xy and the offsets (then `xy` / `off` above point at those outputs)
  const unsigned short* ph;
  const unsigned char* pvl;
  const short* pst;
  const unsigned short* pu;
  const long long* pb;
};
static_assert(kRpBlock == 2 * kPrepPolys, "a prep tile is half a packed block");
struct PrepArgs {
  PrepSet set[kPrepMaxSets];
  int64_t tile_end[kPrepMaxSets];  // exclusive prefix ends of the sets' tile ranges
  int nsets;
  int validate;
  int packed;  // sccg_prep_sets_packed
  unsigned long long* ticket;
};

// Block reduction of a CTA's statistics, then one atomic per field.
__device__ void flush_stats(StatAcc& acc, SetStats* stats, unsigned long long* s_acc, int* s_b) {
  const int lane = threadIdx.x & 31;
  __syncthreads();
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s_b[0] = s_b[1] = INT_MAX;
    s_b[2] = s_b[3] = INT_MIN;
    s_b[4] = s_b[5] = 0;
  }
  __syncthreads();
  unsigned long long v[4] = {acc.nonempty, acc.sw, acc.sh, acc.swh};
  for (int f = 0; f < 4; f++) {
    unsigned long long x = v[f];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && x) atomicAdd(&s_acc[f], x);
  }
  const int bx0 = __reduce_min_sync(0xffffffffu, acc.bx0), by0 = __reduce_min_sync(0xffffffffu, acc.by0);
  const int bx1 = __reduce_max_sync(0xffffffffu, acc.bx1), by1 = __reduce_max_sync(0xffffffffu, acc.by1);
  const int mw = __reduce_max_sync(0xffffffffu, acc.mw), mh = __reduce_max_sync(0xffffffffu, acc.mh);
  if (lane == 0) {
    atomicMin(&s_b[0], bx0);
    atomicMin(&s_b[1], by0);
    atomicMax(&s_b[2], bx1);
    atomicMax(&s_b[3], by1);
    atomicMax(&s_b[4], mw);
    atomicMax(&s_b[5], mh);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_acc[0]) {
    atomicAdd(&stats->nonempty, s_acc[0]);
    atomicAdd(&stats->sw, s_acc[1]);
    atomicAdd(&stats->sh, s_acc[2]);
    atomicAdd(&stats->swh, s_acc[3]);
    atomicMin(&stats->bounds[0], s_b[0]);
    atomicMin(&stats->bounds[1], s_b[1]);
    atomicMax(&stats->bounds[2], s_b[2]);
    atomicMax(&stats->bounds[3], s_b[3]);
    atomicMax(&stats->maxext[0], s_b[4]);
    atomicMax(&stats->maxext[1], s_b[5]);
  }
  acc.init();
}

#ifndef SCCG_PREP_MINB
#define SCCG_PREP_MINB (640 / SCCG_PREP_THREADS)  // 5 CTAs of 128 threads per SM (shared memory)
#endif
template <bool PK>
__global__ void __launch_bounds__(kPrepThreads, SCCG_PREP_MINB) prep_kernel(const __grid_constant__ PrepArgs args) {
  pdl_entry_deferred();  // prep_init's counters
  extern __shared__ int4 s_dyn4[];  // kPrepVerts int2 (16-byte aligned)
  int2* s_xy = reinterpret_cast<int2*>(s_dyn4);
  __shared__ int64_t s_off[kPrepPolys + 1];
  __shared__ unsigned s_big[kPrepPolys / 32];
  __shared__ int s_cnt[kSortKeys];
  __shared__ unsigned char s_perm[kPrepPolys];
  __shared__ unsigned long long s_acc[4];
  __shared__ int s_b[6];
  __shared__ uint64_t s_bar;
  __shared__ long long s_tile;
  __shared__ int s_pk[2][kPrepThreads / 32 + 1];  // packed mode: per-warp scan totals, then the first half's
  __shared__ int s_uoff[kPrepPolys];                // packed mode: each ring's first move unit (block-relative)
  __shared__ int s_uend;                            // packed mode: the tile's end unit (block-relative)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned phase = 0;
  if (threadIdx.x == 0) mbar_init(&s_bar);
  StatAcc acc;
  acc.init();
  const int validate = args.validate;
  const int64_t ntiles = args.tile_end[args.nsets - 1];
  // Tile gt's polygon range (set, first polygon, count) and the offsets this
  // thread stages for it (offsets[p0 + t], thread 0 also offsets[p0 + np]):
  // fetched one tile ahead, so their round trips overlap the current tile.
  auto tile_range = [&](int64_t g, int& si, int64_t& p0, int& np) {
    si = 0;
    while (g >= args.tile_end[si]) si++;
    p0 = (g - (si ? args.tile_end[si - 1] : 0)) * kPrepPolys;
    np = (int)min((int64_t)kPrepPolys, args.set[si].n - p0);
  };
  int64_t off_a = 0, off_b = 0;
  auto fetch_offsets = [&](int64_t g) {
    if (PK || g >= ntiles) return;
    int si2, np2;
    int64_t p02;
    tile_range(g, si2, p02, np2);
    const int64_t* o = args.set[si2].off;
    if ((int)threadIdx.x <= np2) off_a = o[p02 + threadIdx.x];
    if (threadIdx.x == 0) off_b = o[p02 + np2];
  };
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(args.ticket, 1ull);
  __syncthreads();
  int64_t gt = s_tile;
  fetch_offsets(gt);
  int cur = -1;  // set of the statistics in acc
  for (;;) {
    if (gt >= ntiles) break;
    int si;
    int64_t p0;
    int np;
    tile_range(gt, si, p0, np);
    if (si != cur) {
      if (cur >= 0) flush_stats(acc, args.set[cur].stats, s_acc, s_b);
      cur = si;
    }
    const PrepSet& S = args.set[si];
    const int2* __restrict__ xy = S.xy;
    const int64_t nv_total = S.nv_total;
    int4* __restrict__ mbr = S.mbr;
    int64_t* __restrict__ area = S.area;
    int2* __restrict__ ecount = S.ecount;
    uint64_t* __restrict__ edges = S.edges;
    uint32_t* __restrict__ status = S.status;
    const int bulk = S.bulk;
    // the previous tile's bulk write-back must have read the buffer before anything (TMA load or, for a set
    // without 16-byte alignment, plain stores) overwrites it -- whatever the current set's mode
#if SCCG_PREP_USED_ONLY
    bulk_store_drain();  // this thread's write-backs of the previous tile have read the buffer
#else
    if (threadIdx.x == 0) bulk_store_drain();
#endif
    __syncthreads();  // previous tile's shared data fully consumed
    int pk_h = 0, pk_x = 0, pk_y = 0;  // packed mode: this thread's ring head and start
    if (PK) {
      // the tile is half of packed block b: the block scan of (vertices,
      // units) over its 256 heads gives this half's offsets
      const int64_t bb = p0 / kRpBlock;
      const int half = (int)((p0 / kPrepPolys) & 1);
      const long long* blk = args.set[si].pb + 4 * bb;
      const long long vbase = blk[0], sw = blk[2], org = blk[3];
      const int64_t r0 = bb * kRpBlock + threadIdx.x, r1 = r0 + kPrepPolys;
      auto vu = [&](int64_t r, int& V, int& nu, int& h) {
        V = nu = h = 0;
        if (r < args.set[si].n) {
          h = args.set[si].ph[r];
          V = h & 0x1fff;
          const int w = (h >> 13) & 3;
          nu = w == 3 ? (int)args.set[si].pvl[r] : rp_units(max(V - 1, 0), w);
        }
      };
      int Va, nua, ha, Vb, nub, hb;
      vu(r0, Va, nua, ha);
      vu(r1, Vb, nub, hb);
      // first half's totals (needed by the second half), and this half's scan
      int ta = Va, tu = nua, xv = half ? Vb : Va, xu = half ? nub : nua;
      for (int o = 16; o; o >>= 1) {
        ta += __shfl_xor_sync(0xffffffffu, ta, o);
        tu += __shfl_xor_sync(0xffffffffu, tu, o);
      }
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, xv, o), c = __shfl_up_sync(0xffffffffu, xu, o);
        if (lane >= o) {
          xv += a;
          xu += c;
        }
      }
      if (lane == 31) {
        s_pk[0][warp] = xv;
        s_pk[1][warp] = xu;
      }
      if (lane == 0) {
        s_cnt[2 * warp] = ta;  // (s_cnt is cleared below, after use)
        s_cnt[2 * warp + 1] = tu;
      }
      __syncthreads();
      int bv = 0, bu = 0, fv = 0, fu = 0;
      for (int w2 = 0; w2 < kPrepThreads / 32; w2++) {
        bv += w2 < warp ? s_pk[0][w2] : 0;
        bu += w2 < warp ? s_pk[1][w2] : 0;
        fv += s_cnt[2 * w2];
        fu += s_cnt[2 * w2 + 1];
      }
      const int myV = half ? Vb : Va, mynu = half ? nub : nua;
      const int vpre = bv + xv - myV + (half ? fv : 0), upre = bu + xu - mynu + (half ? fu : 0);
      pk_h = half ? hb : ha;
      if ((int)threadIdx.x < np) {
        s_off[threadIdx.x] = vbase + vpre;
        s_uoff[threadIdx.x] = upre;
        if ((int)threadIdx.x == np - 1) {
          s_off[np] = vbase + vpre + myV;
          s_uend = upre + mynu;
        }
        // start of this thread's ring (narrow block: int16 deltas from the block origin)
        const int jb = half * kPrepPolys + threadIdx.x;
        const long long so = sw & ((1ll << 62) - 1);
        if ((sw >> 62) & 1) {
          const unsigned short* sp = reinterpret_cast<const unsigned short*>(args.set[si].pst) + so + 4 * jb;
          pk_x = (int)((unsigned)sp[0] | ((unsigned)sp[1] << 16));
          pk_y = (int)((unsigned)sp[2] | ((unsigned)sp[3] << 16));
        } else {
          pk_x = (int)(unsigned)(org & 0xffffffffll) + args.set[si].pst[so + 2 * jb];
          pk_y = (int)(unsigned)((unsigned long long)org >> 32) + args.set[si].pst[so + 2 * jb + 1];
        }
      }
      __syncthreads();  // s_cnt / s_pk reused below
      if ((int)threadIdx.x < np) {  // the offsets are an output of packed mode
        int64_t* oo = const_cast<int64_t*>(args.set[si].off);
        oo[p0 + threadIdx.x] = s_off[threadIdx.x];
        if (p0 + np == args.set[si].n && (int)threadIdx.x == np - 1) oo[p0 + np] = s_off[np];
      }
    } else {
      if ((int)threadIdx.x <= np) s_off[threadIdx.x] = off_a;
      if (threadIdx.x == 0) s_off[np] = off_b;
    }
    long long next_gt = 0;
    if (threadIdx.x == 0) next_gt = (long long)atomicAdd(args.ticket, 1ull);  // the next tile, in flight
    if (threadIdx.x < kPrepPolys / 32) s_big[threadIdx.x] = 0;
    for (int t = threadIdx.x; t < kSortKeys; t += kPrepThreads) s_cnt[t] = 0;
    s_perm[threadIdx.x] = 0xff;
    // packed mode: the tile's move units staged in the free tail of the tile buffer (when the decoded
    // vertices leave room), so each thread's bit-window refills are shared-memory loads
    const unsigned short* pk_units = nullptr;
    if (PK) {
      const unsigned short* gu = args.set[si].pu + args.set[si].pb[4 * (p0 / kRpBlock) + 1];
      const int u0 = np > 0 ? s_uoff[0] : 0, nunits = np > 0 ? s_uend - u0 : 0;
      const int64_t tv0 = s_off[0] & ~int64_t(1), tnv = s_off[np] - tv0;
      const int ubytes = (2 * nunits + 15) & ~15;
      if (tnv >= 0 && tnv * 8 + ubytes <= (int64_t)kPrepSmem) {
        unsigned short* su = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(s_dyn4) + kPrepSmem - ubytes);
        for (int i = threadIdx.x; i < nunits; i += kPrepThreads) su[i] = __ldg(gu + u0 + i);
        pk_units = su - u0;  // indexed by block-relative unit
      } else {
        pk_units = gu;
      }
    }
    __syncthreads();
    // Rings are dealt to threads in order of vertex count (counting sort on
    // V / 4), so the lanes of a warp run loops of similar length (dealing them
    // round-robin over the warps instead balances the warps but costs ~30%
    // more instructions: measured, profiles/r01).
    int key = 0, pos = 0;
    if (threadIdx.x < np) {
      key = (int)min((s_off[threadIdx.x + 1] - s_off[threadIdx.x]) >> SCCG_PREP_SORT_SHIFT, (int64_t)kSortKeys - 1);
      key = max(key, 0);
      pos = atomicAdd(&s_cnt[key], 1);
    }
    // stage the tile's vertex range [v0, v1) (v0 even): one TMA bulk copy of the
    // 16-byte-aligned body, the odd last vertex by a thread
    const int64_t v0 = s_off[0] & ~int64_t(1), v1 = s_off[np];
    const bool tiled = s_off[0] >= 0 && v1 <= nv_total && v1 >= s_off[0] && v1 - v0 <= kPrepVerts;
    if (PK) {
      // (decoded below, after the rings are dealt by length)
    } else if (tiled) {
      const int64_t nv = v1 - v0;
      if (bulk) {
        if (threadIdx.x == 0) {
          bulk_store_drain();  // the previous tile's write-back has read the buffer
          fence_async_smem();
          if (nv >= 2) bulk_load(s_dyn4, xy + v0, (unsigned)(nv >> 1) * 16u, &s_bar);
          if (nv & 1) s_xy[nv - 1] = xy[v1 - 1];
        }
        if (nv >= 2) {
          mbar_wait(&s_bar, phase);
          phase ^= 1u;
        }
      } else {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) s_xy[i] = xy[v0 + i];
      }
    }
    __syncthreads();  // every ring counted (packed mode: every ring decoded)
    if (threadIdx.x < 32) {  // exclusive scan of the bucket counts (two per lane)
      const int c0 = s_cnt[2 * threadIdx.x], c1 = s_cnt[2 * threadIdx.x + 1];
      int incl = c0 + c1;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)threadIdx.x >= o) incl += t;
      }
      s_cnt[2 * threadIdx.x] = incl - c0 - c1;
      s_cnt[2 * threadIdx.x + 1] = incl - c1;
    }
    __syncthreads();
    if (threadIdx.x < np) s_perm[s_cnt[key] + pos] = (unsigned char)threadIdx.x;
    __syncthreads();
#if SCCG_PREP_RES_DEAL == 2
    // Within each warp's 32 rings (similar lengths, from the sort above), deal
    // the rings to the two half-warps so that each half's rings start at
    // distinct shared-memory bank pairs as far as possible (residue = (offset
    // - v0) mod 16 vertices = 128 bytes; a half-warp's lockstep 8-byte reads of
    // vertex i of 16 rings are one wavefront when the residues differ): the
    // occurrences of each residue alternate between the halves, and the halves
    // are evened out by moving the last occurrence of half of the residues
    // that occur an odd number of times.  A residue occurring c times costs
    // ceil(c / 2) wavefronts per half instead of up to c.
    {
      const int j = s_perm[threadIdx.x];
      const int res = j != 0xff ? (int)((s_off[j] - v0) & 15) : 16 + (lane & 15);
      const unsigned peers = __match_any_sync(0xffffffffu, res);
      const int o = __popc(peers & lanemask_lt()), c = __popc(peers);
      int half = o & 1;
      const bool cand = (c & 1) && o == c - 1;  // the extra occurrence of an odd count (in half 0)
      const unsigned cm = __ballot_sync(0xffffffffu, cand);
      if (cand && __popc(cm & lanemask_lt()) < (__popc(cm) >> 1)) half = 1;
      const unsigned hm = __ballot_sync(0xffffffffu, half == 1);
      const int pos = __popc((half ? hm : ~hm) & lanemask_lt());
      __syncwarp();
      s_perm[warp * 32 + half * 16 + pos] = (unsigned char)j;
      __syncthreads();
    }
#elif SCCG_PREP_RES_DEAL == 1
    // Within each warp's 32 rings (similar lengths, from the sort above), deal
    // the rings to lanes by the shared-memory bank of their first vertex
    // ((offset - v0) mod 16 vertices = 128 bytes): rings sorted by that residue
    // go alternately to the two half-warps, so a half-warp's lockstep reads of
    // vertex i of 16 rings mostly hit distinct bank pairs in the edge pass.
    {
      const int j = s_perm[threadIdx.x];
      const int res = j != 0xff ? (int)((s_off[j] - v0) & 15) : 16;
      int rank = 0;
      for (int l = 0; l < 32; l++) {
        const int rl = __shfl_sync(0xffffffffu, res, l);
        rank += (rl < res || (rl == res && l < lane)) ? 1 : 0;
      }
      __syncwarp();
      s_perm[warp * 32 + (rank & 1) * 16 + (rank >> 1)] = (unsigned char)j;
      __syncthreads();
    }
#endif
    if (PK) {
      // decode the ring this thread was dealt (by length: a warp's serial
      // walks have similar trip counts) into the tile -- or, for a tile too
      // large to stage, straight into xy -- then the tile goes to xy by one
      // bulk store, read out before the ring work rewrites it in place
      const int j = s_perm[threadIdx.x];
      if (j != 0xff) {
        const int64_t r = p0 + j;
        const int hj = args.set[si].ph[r], V = hj & 0x1fff;
        const int64_t rb = s_off[j];
        if (V > 0 && rb >= 0 && rb + V <= nv_total) {  // (an encoding inconsistent with n_vertices writes nothing)
          const long long* blk = args.set[si].pb + 4 * (p0 / kRpBlock);
          const long long sw = blk[2], org = blk[3], so = sw & ((1ll << 62) - 1);
          const int jb = (int)(r - (p0 / kRpBlock) * kRpBlock);
          int x, y;
          if ((sw >> 62) & 1) {
            const unsigned short* sp = reinterpret_cast<const unsigned short*>(args.set[si].pst) + so + 4 * jb;
            x = (int)((unsigned)sp[0] | ((unsigned)sp[1] << 16));
            y = (int)((unsigned)sp[2] | ((unsigned)sp[3] << 16));
          } else {
            x = (int)(unsigned)(org & 0xffffffffll) + args.set[si].pst[so + 2 * jb];
            y = (int)(unsigned)((unsigned long long)org >> 32) + args.set[si].pst[so + 2 * jb + 1];
          }
          int2* dst = tiled ? s_xy + (rb - v0) : const_cast<int2*>(xy) + rb;
          rp_walk_ring(pk_units + s_uoff[j], V, (hj >> 13) & 3, hj >> 15, x, y, dst);
        }
      }
      fence_async_smem();  // this thread's decoded vertices -> async proxy (the bulk store below)
      __syncthreads();
      if (tiled) {  // the decoded tile [off[p0], v1) -> xy
        const int64_t s0 = s_off[0];
        const int64_t a0 = (s0 + 1) & ~int64_t(1), a1 = v1 & ~int64_t(1);
        int2* xo = const_cast<int2*>(xy);
        if (bulk) {
          if (threadIdx.x == 0) {
            if (a1 > a0) bulk_store(xo + a0, s_xy + (a0 - v0), (unsigned)(a1 - a0) * 8u);
            if (s0 < a0 && s0 < v1) xo[s0] = s_xy[s0 - v0];
            if (a1 < v1 && a1 >= a0) xo[a1] = s_xy[a1 - v0];
            bulk_store_drain();  // read out of shared memory before anyone rewrites it
          }
        } else {
          for (int64_t i = s0 + threadIdx.x; i < v1; i += blockDim.x) xo[i] = s_xy[i - v0];
        }
      }
      __syncthreads();
    }
#if SCCG_PREP_L2_PREFETCH == 2
    if (!PK && threadIdx.x == 0) {
      // thread 0 (warp 0 deals the smallest rings, so it has slack) starts
      // pulling the next tile's vertex range into L2 while this tile's rings
      // are worked on: that tile's TMA load then hits L2 instead of HBM
      // (also prefetching the tile one grid-width further measured slower: 161 vs 159 us)
      auto prefetch_tile = [&](long long g) {
        if (g >= ntiles) return;
        int si2, np2;
        int64_t p02;
        tile_range(g, si2, p02, np2);
        const PrepSet& S2 = args.set[si2];
        if (!S2.bulk) return;
        const int64_t w0 = S2.off[p02] & ~int64_t(1), w1 = S2.off[p02 + np2];
        if (w0 >= 0 && w1 > w0 && w1 <= S2.nv_total && w1 - w0 <= kPrepVerts) {
          const unsigned bytes = (unsigned)((w1 - w0 + 1) & ~int64_t(1)) * 8u;
          prefetch_l2(S2.xy + w0, bytes);
        }
      };
      prefetch_tile(next_gt);
    }
#endif
    // thread per small ring (records in place in the tile)
    if (s_perm[threadIdx.x] != 0xff) {
      const int j = s_perm[threadIdx.x];
      const int64_t poly = p0 + j;
      const int64_t b = s_off[j], e = s_off[j + 1];
      const int64_t V = e - b;
      if (b < 0 || e > nv_total || V < 4) {  // malformed offsets or too few vertices
        mbr[poly] = make_int4(0, 0, 0, 0);
        area[poly] = 0;
        ecount[poly] = make_int2(0, 0);
        flag(status, SCCG_STATUS_ARG, poly);
      } else if (V > kThreadMaxV || !tiled) {
        atomicOr(&s_big[j >> 5], 1u << (j & 31));
      } else {
        int used8;
        const int rot = (int)((lane - (b - v0)) & 15);  // raster pass: record rot first (bank pairs by lane)
        acc.add(prep_polygon_thread(s_xy + (b - v0), (int)V, rot, poly, mbr, area, ecount, status, validate, used8));
#if SCCG_PREP_USED_ONLY
        if (bulk) store_used(edges, b, reinterpret_cast<const uint64_t*>(s_xy + (b - v0)), used8);
        else
          for (int i = 0; i < used8; i++) edges[b + i] = reinterpret_cast<const uint64_t*>(s_xy + (b - v0))[i];
#endif
      }
    }
    if (threadIdx.x == 0) {
      s_tile = next_gt;
#if SCCG_PREP_L2_PREFETCH == 1
      // warp 0 deals the smallest rings and waits here for the others: its
      // lane 0 starts pulling the next tile's vertex range into L2, so that
      // tile's TMA load hits L2 instead of HBM
      if (next_gt < ntiles) {
        int si2, np2;
        int64_t p02;
        tile_range(next_gt, si2, p02, np2);
        const PrepSet& S2 = args.set[si2];
        if (S2.bulk) {
          const int64_t w0 = S2.off[p02] & ~int64_t(1), w1 = S2.off[p02 + np2];
          if (w0 >= 0 && w1 > w0 && w1 <= S2.nv_total && w1 - w0 <= kPrepVerts) {
            const unsigned bytes = (unsigned)((w1 - w0 + 1) & ~int64_t(1)) * 8u;
            prefetch_l2(S2.xy + w0, bytes);
          }
        }
      }
#endif
    }
    __syncthreads();
    const int64_t gt_next = s_tile;
    fetch_offsets(gt_next);  // in flight during the rest of this tile
    // warp per large ring (in the tile when tiled, else straight from global)
    for (int w = 0; w < kPrepPolys / 32; w++) {
      unsigned bits = s_big[w];
      for (int t = 0; bits; t++) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1;
        if ((t & (kPrepThreads / 32 - 1)) != warp) continue;
        const int j = w * 32 + bit;
        const int64_t poly = p0 + j;
        const int64_t b = s_off[j], e = s_off[j + 1];
        int2* src = tiled ? s_xy + (b - v0) : const_cast<int2*>(xy) + b;
        uint64_t* out = tiled ? reinterpret_cast<uint64_t*>(src) : edges + b;
        int nv;
        const int4 m = prep_polygon(src, e - b, poly, out, mbr, area, ecount, status, validate, tiled, nv);
        if (lane == 0) acc.add(m);
#if SCCG_PREP_USED_ONLY
        if (tiled) {  // records are in the tile: write them back
          __syncwarp();
          if (bulk) {
            fence_async_smem();
            __syncwarp();
            if (lane == 0) store_used(edges, b, out, nv);
          } else {
            for (int i = lane; i < nv; i += 32) edges[b + i] = out[i];
          }
        }
#endif
      }
    }
    __syncthreads();
    // write-back of the tile's slots [off[p0], v1) -- exactly this tile's rings
    // (v0 may be the previous tile's last slot): one TMA bulk store of the
    // 16-byte-aligned body, the odd ends by a thread
    if (tiled && !SCCG_PREP_USED_ONLY) {
      const int64_t s0 = s_off[0];
      const int64_t a0 = (s0 + 1) & ~int64_t(1), a1 = v1 & ~int64_t(1);
      const uint64_t* rec = reinterpret_cast<const uint64_t*>(s_xy);
      if (bulk) {
        fence_async_smem();  // this thread's shared-memory records -> async proxy
        __syncthreads();
        if (threadIdx.x == 0) {
          if (a1 > a0) bulk_store(edges + a0, rec + (a0 - v0), (unsigned)(a1 - a0) * 8u);
          if (s0 < a0 && s0 < v1) edges[s0] = rec[s0 - v0];
          if (a1 < v1 && a1 >= a0) edges[a1] = rec[a1 - v0];
        }
      } else {
        for (int64_t i = s0 + threadIdx.x; i < v1; i += blockDim.x) edges[i] = rec[i - v0];
      }
    }
    gt = gt_next;
  }
  pdl_done();  // no tile left: the join's first kernel may launch
  if (SCCG_PREP_USED_ONLY || threadIdx.x == 0) bulk_store_drain();  // shared memory must outlive the write-backs
  if (cur >= 0) flush_stats(acc, args.set[cur].stats, s_acc, s_b);
}

__global__ void prep_init_kernel(PrepArgs args) {
  pdl_trigger();
  const int i = threadIdx.x;
  if (i < args.nsets) {
    uint32_t* status = args.set[i].status;
    SetStats* st = args.set[i].stats;
    status[0] = 0;
    status[1] = 0xffffffffu;
    st->bounds[0] = st->bounds[1] = INT_MAX;
    st->bounds[2] = st->bounds[3] = INT_MIN;
    st->maxext[0] = st->maxext[1] = 0;
    st->pad[0] = st->pad[1] = 0;
    st->nonempty = st->sw = st->sh = st->swh = 0;
  }
  if (args.packed && i < args.nsets && args.set[i].n == 0)  // packed mode, no rings: offsets[0]
    const_cast<int64_t*>(args.set[i].off)[0] = 0;
  if (i == 0) *args.ticket = 0;
}

cudaError_t launch_prep(const sccg_polyset* const* sets, int count, int validate, cudaStream_t st,
                        const sccg_rect_packed* pk) {
  PrepArgs a{};
  a.packed = pk ? 1 : 0;
  a.nsets = count;
  a.validate = validate;
  int64_t tiles = 0;
  for (int i = 0; i < count; i++) {
    const sccg_polyset* s = sets[i];
    PrepSet& d = a.set[i];
    d.xy = reinterpret_cast<const int2*>(s->xy);
    d.off = s->offsets;
    d.n = s->n_polygons;
    d.nv_total = s->n_vertices;
    d.mbr = reinterpret_cast<int4*>(s->mbr);
    d.area = s->area;
    d.ecount = reinterpret_cast<int2*>(s->ecount);
    d.edges = s->edges;
    d.status = s->status;
    d.stats = reinterpret_cast<SetStats*>(s->stats);
    d.bulk = ((reinterpret_cast<uintptr_t>(s->xy) | reinterpret_cast<uintptr_t>(s->edges)) & 15) == 0 ? 1 : 0;
#ifdef SCCG_PREP_NO_TMA  // ablation build (scripts/fig9.py): tiles staged by plain LSU copies
    d.bulk = 0;
#endif
    if (pk) {
      d.ph = pk[i].head;
      d.pvl = pk[i].vlen;
      d.pst = pk[i].start;
      d.pu = pk[i].units;
      d.pb = reinterpret_cast<const long long*>(pk[i].block);
    }
    tiles += (s->n_polygons + kPrepPolys - 1) / kPrepPolys;
    a.tile_end[i] = tiles;
  }
  // the ticket lives in the first set's statistics block (reserved words)
  a.ticket = &reinterpret_cast<SetStats*>(sets[0]->stats)->reserved[0];
  prep_init_kernel<<<1, 32, 0, st>>>(a);
  if (tiles > 0) {
    static cudaError_t attr =
        cudaFuncSetAttribute(prep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPrepSmem);
    static cudaError_t attr_pk =
        cudaFuncSetAttribute(prep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPrepSmem);
    if (attr != cudaSuccess) return attr;
    if (attr_pk != cudaSuccess) return attr_pk;
    static int sms = 0, per_sm = 1;
    if (sms == 0) {  // launch geometry, queried once per process
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep_kernel<false>, kPrepThreads, kPrepSmem);
    }
    int64_t blocks = tiles;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    if (cudaError_t e = pk ? launch_pdl(prep_kernel<true>, dim3((unsigned)blocks), dim3(kPrepThreads), kPrepSmem, st, a)
                           : launch_pdl(prep_kernel<false>, dim3((unsigned)blocks), dim3(kPrepThreads), kPrepSmem, st,
                                        a))
      return e;
  }
  return cudaGetLastError();
}

}  // namespace sccg
