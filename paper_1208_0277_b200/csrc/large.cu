// large.cu -- PixelBox for large pairs:
// region work items with local edge culling.
//
// Every pair the small kernel cannot take (root box wider or taller than 32,
// |box| >= T, or rings with more than 64 vertical edges) lands here.
//  1. (in the small kernel, emit_large) the pair's root box MBR(p) n MBR(q)
//     (reading R5) is cut into up to 32 x 32 disjoint regions of about
//     128 x 128 pixels -- the "huge-pair split into region work items" of
//     so one large pair is spread over many warps (the paper
//     gives a whole pair to one block, which leaves a few big pairs on
//     a few SMs).
//  2. item_kernel: a warp takes one item (pair, region R) from a global queue:
//     - it culls both polygons' edges to those meeting R (vertical edges with
//       x strictly inside R's columns, horizontal edges strictly inside R's
//       rows -- all other edges cannot reach R's open interior) into shared
//       memory, and casts one ray for R's corner pixel;
//     - it then runs Algorithm 1 on R with a warp-private DFS stack
//       of sampling boxes.  Lemma 1 (reading R6-A) classifies the <= 32 aligned
//       sub-boxes of a split edge-parallel (a lane owns an edge, the warp
//       OR/XOR-reduces 32-bit sub-box masks); a sub-box corner's parity is its
//       parent corner's parity plus the crossings along the parent's left
//       column and the sub-box's bottom row, so only local edges are touched;
//     - boxes below T are pixelized bit-parallel (a lane owns a 32-pixel row
//       word: row parity at the box's left column, then one suffix mask per
//       local vertical edge);
//     - the item's pixel count is added into the pair's int64 accumulator;
//       the warp finishing a pair's last item finalizes the pair: U = |p| +
//       |q| - I, the outputs, the exact totals (reading R12).
//     An item whose local lists overflow shared memory is split in two and
//     retried (in the same warp), so any input is handled.
// Regions are disjoint and cover the root box exactly, so the per-pair sums are
// exact and independent of the split (integer atomics are order-free).
#include "pixelbox_common.cuh"

namespace sccg {

#ifndef SCCG_DENSE_SPLIT
#define SCCG_DENSE_SPLIT 1
#endif
#ifndef SCCG_DENSE_NUM  // a split is dense when more than NUM/DEN of its sub-boxes hover (1/4: measured best
#define SCCG_DENSE_NUM 1   // of 1/4, 1/2, 3/4 on C3 and C5)
#define SCCG_DENSE_DEN 4
#endif
constexpr int kLWarps = 4;          // warps per CTA
constexpr int kLCap = 192;          // local records per list (vertical / horizontal) per polygon per warp
constexpr int kLStage = 96;         // staged records per polygon for one pixelized box
constexpr int kLStack = 256;        // sampling boxes per warp stack
constexpr int kLItems = 48;         // in-warp item stack (overflow splits)

struct PolyRef {
  const uint64_t* ev;  // vertical records (decode_edge with o0: relative to the polygon MBR origin)
  unsigned o0;         // the records' rebase (ecount.y)
  const int2* v;       // raw ring (horizontal edges)
  int nv, V;
  int dx, dy;          // polygon MBR origin - root-box origin
  int ox, oy;          // root-box origin (absolute)
};

// packed local records (relative to the item region origin, clamped so all
// comparisons against boxes inside the region are preserved):
//   vertical:   x (15 bit, 0 < x < Wr), ylo, yhi (int16, in [-1, Hr + 1])
//   horizontal: y (15 bit, 0 < y < Hr), xlo, xhi (int16, in [-1, Wr + 1])
__device__ __forceinline__ uint64_t pack_loc(int a, int lo, int hi) {
  return (uint64_t)(uint32_t)(a & 0xffff) | ((uint64_t)(uint32_t)(lo & 0xffff) << 16) |
         ((uint64_t)(uint32_t)(hi & 0xffff) << 32);
}
__device__ __forceinline__ void unpack_loc(uint64_t r, int& a, int& lo, int& hi) {
  a = (int)(r & 0xffff);
  lo = (int)(short)((r >> 16) & 0xffff);
  hi = (int)(short)((r >> 32) & 0xffff);
}

struct LocalPoly {
  uint64_t* V;  // [kLCap]
  uint64_t* H;  // [kLCap]
  int nV, nH;
  int pi;       // parity of the region's corner pixel (1 = inside)
};

#ifndef SCCG_CULL_GROUPS
#define SCCG_CULL_GROUPS 4
#endif
constexpr int kCullGroups = SCCG_CULL_GROUPS;  // 32-wide load groups in flight in the culling loops

// Cull one polygon's edges to region R = [X0, X1) x [Y0, Y1) (root coords)
// and cast the corner ray.  Returns false if a list overflows.
__device__ bool build_local(const PolyRef& c, int X0, int Y0, int X1, int Y1, LocalPoly& L) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int Wr = X1 - X0, Hr = Y1 - Y0;
  int par = 0, cnt = 0;
  // records / vertices are read four 32-wide groups at a time (all loads in
  // flight before any is used: this culling re-reads both rings per region
  // item, and on comb pairs it is the kernel's main memory stall)
  for (int j00 = 0; j00 < c.nv; j00 += 32 * kCullGroups) {
    uint64_t rr[kCullGroups];
#pragma unroll
    for (int u = 0; u < kCullGroups; u++) {
      const int j = j00 + 32 * u + lane;
      rr[u] = j < c.nv ? __ldg(c.ev + j) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kCullGroups; u++) {
      const int j0 = j00 + 32 * u;
      if (j0 >= c.nv) break;  // warp-uniform
      const int j = j0 + lane;
      bool keep = false;
      uint64_t rec = 0;
      if (j < c.nv) {
        int cc, lo, hi;
        decode_edge(rr[u], c.o0, cc, lo, hi);
        const int x = cc + c.dx, yl = lo + c.dy, yh = hi + c.dy;
        par ^= (x > X0 && yl <= Y0 && Y0 < yh) ? 1 : 0;  // ray from (X0 + 1/2, Y0 + 1/2) toward +x
        keep = x > X0 && x < X1 && yl < Y1 && yh > Y0;
        rec = pack_loc(x - X0, max(yl - Y0, -1), min(yh - Y0, Hr + 1));
      }
      const unsigned b = __ballot_sync(FULL, keep);
      const int pos = cnt + __popc(b & lt);
      if (keep && pos < kLCap) L.V[pos] = rec;
      cnt += __popc(b);
    }
  }
  L.nV = cnt;
  L.pi = __reduce_xor_sync(FULL, (unsigned)par) & 1;
  cnt = 0;
  const int2 first = c.V > 0 ? __ldg(c.v) : make_int2(0, 0);
  for (int j00 = 0; j00 < c.V; j00 += 32 * kCullGroups) {
    int2 av[kCullGroups];
#pragma unroll
    for (int u = 0; u < kCullGroups; u++) {
      const int j = j00 + 32 * u + lane;
      av[u] = j < c.V ? __ldg(c.v + j) : make_int2(0, 0);
    }
    const int2 tail = j00 + 32 * kCullGroups < c.V ? __ldg(c.v + j00 + 32 * kCullGroups) : first;  // the next block's first
#pragma unroll
    for (int u = 0; u < kCullGroups; u++) {
      const int j0 = j00 + 32 * u;
      if (j0 >= c.V) break;  // warp-uniform
      const int j = j0 + lane;
      // the edge from vertex j to j + 1: the next vertex is the next lane's
      int2 b2;
      b2.x = __shfl_down_sync(FULL, av[u].x, 1);
      b2.y = __shfl_down_sync(FULL, av[u].y, 1);
      const int2 nxt = u < kCullGroups - 1 ? make_int2(__shfl_sync(FULL, av[u < kCullGroups - 1 ? u + 1 : u].x, 0),
                                                       __shfl_sync(FULL, av[u < kCullGroups - 1 ? u + 1 : u].y, 0))
                                           : tail;
      if (lane == 31) b2 = nxt;
      if (j + 1 == c.V) b2 = first;  // the ring closes
      bool keep = false;
      uint64_t rec = 0;
      if (j < c.V) {
        const int2 a = av[u];
        if (a.y == b2.y && a.x != b2.x) {
          const int f = a.y - c.oy, xl = min(a.x, b2.x) - c.ox, xh = max(a.x, b2.x) - c.ox;
          keep = f > Y0 && f < Y1 && xl < X1 && xh > X0;
          rec = pack_loc(f - Y0, max(xl - X0, -1), min(xh - X0, Wr + 1));
        }
      }
      const unsigned b = __ballot_sync(FULL, keep);
      const int pos = cnt + __popc(b & lt);
      if (keep && pos < kLCap) L.H[pos] = rec;
      cnt += __popc(b);
    }
  }
  L.nH = cnt;
  return L.nV <= kLCap && L.nH <= kLCap;
}

// ------------------------------------------------------ per-pair edge index
// build_local streams both whole rings for every region item; a pair cut into
// many regions (a comb, C5; a gland, C3) re-culls its rings once per region,
// which is most of the item kernel's instructions on combs.  So the warp that
// takes a pair's FIRST item (items[0 .. nl) come before every extra item in
// the queue) buckets each ring's vertical edges by region column and its
// horizontal edges by region row -- an edge goes to the column (row) whose
// open interior it lies strictly inside, else to none: then it cannot meet
// any region's open interior -- and computes every region corner's ray parity
// (an XOR difference grid over rows of column masks), into the optional pool.
// The pair's other items cull only their column's and row's buckets.  A
// region's culled lists are the same sets build_local makes (in another
// order; every use of them is order-free), so the areas are unchanged.
#ifndef SCCG_IX_MIN
#define SCCG_IX_MIN 4  // regions per pair worth an index (a build costs two ring passes)
#endif
constexpr int kIxMin = SCCG_IX_MIN;
constexpr int kIxReady = 2, kIxNone = 3;

__device__ __forceinline__ uint64_t pack_ix(int a, int lo, int hi) {
  return (uint64_t)(a & 0x1fffff) | ((uint64_t)(lo & 0x1fffff) << 21) | ((uint64_t)(hi & 0x1fffff) << 42);
}
__device__ __forceinline__ int sx21(uint64_t v) { return ((int)(unsigned)(v & 0x1fffffu) << 11) >> 11; }
__device__ __forceinline__ void unpack_ix(uint64_t r, int& a, int& lo, int& hi) {
  a = sx21(r);
  lo = sx21(r >> 21);
  hi = sx21(r >> 42);
}
// number of the boundaries b[t] = floor(t * L / n), t = 0..n, below the
// integer v: floor(t L / n) < v  <=>  t L / n < v  <=>  t < v n / L, so the
// count is min(n + 1, ceil(v n / L)) for v > 0 (v n < 2^22: 32-bit exact)
__device__ __forceinline__ int count_below(int v, int n, int L) {
  return v <= 0 ? 0 : min(n + 1, (int)(((unsigned)v * (unsigned)n + (unsigned)L - 1u) / (unsigned)L));
}
__device__ __forceinline__ int ld_acquire_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// header words (u32) of one polygon's index: vertical bucket starts [nx + 1],
// horizontal bucket starts [ny + 1] (relative to the horizontal block),
// corner parity masks [ny]; padded to whole 8-byte words
__device__ __forceinline__ int ix_header_words(int nx, int ny) { return (nx + 1 + ny + 1 + ny + 1) / 2; }

// Build pair i's index (one warp).  sc: >= 264 ints of the warp's shared
// scratch.  Returns the pool offset of polygon 0's index, or -1 (no room).
__device__ long long build_index(const PolyRef* pr, int W, int H, int nx, int ny, const LargeWs& w, int* sc) {
  const int lane = threadIdx.x & 31;
  int* X = sc;
  int* Y = sc + 33;
  for (int t = lane; t < 33; t += 32) {
    X[t] = t <= nx ? (int)((long long)t * W / nx) : INT_MAX;
    Y[t] = t <= ny ? (int)((long long)t * H / ny) : INT_MAX;
  }
  for (int t = lane; t < 198; t += 32) sc[66 + t] = 0;
  __syncwarp();
  // pass 1: bucket counts and corner parities
  for (int s = 0; s < 2; s++) {
    const PolyRef& c = pr[s];
    int* cv = sc + 66 + 99 * s;
    int* ch = cv + 33;
    int* D = ch + 33;
    for (int j = lane; j < c.nv; j += 32) {
      int cc, lo, hi;
      decode_edge(__ldg(c.ev + j), c.o0, cc, lo, hi);
      const int x = cc + c.dx, yl = lo + c.dy, yh = hi + c.dy;
      const int cm = count_below(x, nx, W);
      if (cm >= 1 && cm <= nx && X[cm] != x) atomicAdd(&cv[cm - 1], 1);
      const int cols = min(cm, nx);  // corners (X_c, Y_r) whose ray toward +x crosses this edge: X_c < x ...
      const int r0 = min(count_below(yl, ny, H), ny), r1 = min(count_below(yh, ny, H), ny);  // ... and yl <= Y_r < yh
      if (cols > 0 && r0 < r1) {
        atomicXor(reinterpret_cast<unsigned*>(&D[r0]), low_bits(cols));
        atomicXor(reinterpret_cast<unsigned*>(&D[r1]), low_bits(cols));
      }
    }
    for (int j = lane; j < c.V; j += 32) {
      const int2 a = __ldg(c.v + j), b = __ldg(c.v + (j + 1 == c.V ? 0 : j + 1));
      if (a.y == b.y && a.x != b.x) {
        const int f = a.y - c.oy;
        const int rm = count_below(f, ny, H);
        if (rm >= 1 && rm <= ny && Y[rm] != f) atomicAdd(&ch[rm - 1], 1);
      }
    }
  }
  __syncwarp();
  // bucket starts (exclusive scans over <= 32 buckets), parities (prefix XOR)
  int totv[2], toth[2];
  for (int s = 0; s < 2; s++) {
    int* cv = sc + 66 + 99 * s;
    int* ch = cv + 33;
    int* D = ch + 33;
    int v = lane < nx ? cv[lane] : 0, h = lane < ny ? ch[lane] : 0;
    unsigned d = lane < ny ? (unsigned)D[lane] : 0u;
    int iv = v, ih = h;
    unsigned id = d;
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(FULL, iv, o), b = __shfl_up_sync(FULL, ih, o);
      const unsigned e = __shfl_up_sync(FULL, id, o);
      if (lane >= o) {
        iv += a;
        ih += b;
        id ^= e;
      }
    }
    totv[s] = __shfl_sync(FULL, iv, 31);
    toth[s] = __shfl_sync(FULL, ih, 31);
    __syncwarp();
    if (lane < nx) cv[lane] = iv - v;
    if (lane < ny) {
      ch[lane] = ih - h;
      D[lane] = (int)id;
    }
    __syncwarp();
  }
  const int hw = ix_header_words(nx, ny);
  const long long need0 = hw + totv[0] + toth[0], need = need0 + hw + totv[1] + toth[1];
  long long base = 0;
  if (lane == 0) base = (long long)atomicAdd(&w.ctr[3], (unsigned long long)need);
  base = __shfl_sync(FULL, base, 0);
  if (base + need > w.pool_cap) return -1;
  // headers, then the records (pass 2, each to its bucket's next slot)
  for (int s = 0; s < 2; s++) {
    const PolyRef& c = pr[s];
    int* cv = sc + 66 + 99 * s;
    int* ch = cv + 33;
    const int* D = ch + 33;
    uint64_t* blk = w.pool + base + (s ? need0 : 0);
    unsigned* hdr = reinterpret_cast<unsigned*>(blk);
    for (int t = lane; t <= nx; t += 32) hdr[t] = t < nx ? (unsigned)cv[t] : (unsigned)totv[s];
    for (int t = lane; t <= ny; t += 32) hdr[nx + 1 + t] = t < ny ? (unsigned)ch[t] : (unsigned)toth[s];
    for (int t = lane; t < ny; t += 32) hdr[nx + ny + 2 + t] = (unsigned)D[t];
    uint64_t* vrec = blk + hw;
    uint64_t* hrec = vrec + totv[s];
    for (int j = lane; j < c.nv; j += 32) {
      int cc, lo, hi;
      decode_edge(__ldg(c.ev + j), c.o0, cc, lo, hi);
      const int x = cc + c.dx, yl = lo + c.dy, yh = hi + c.dy;
      const int cm = count_below(x, nx, W);
      if (cm >= 1 && cm <= nx && X[cm] != x) vrec[atomicAdd(&cv[cm - 1], 1)] = pack_ix(x, yl, yh);
    }
    for (int j = lane; j < c.V; j += 32) {
      const int2 a = __ldg(c.v + j), b = __ldg(c.v + (j + 1 == c.V ? 0 : j + 1));
      if (a.y == b.y && a.x != b.x) {
        const int f = a.y - c.oy;
        const int rm = count_below(f, ny, H);
        if (rm >= 1 && rm <= ny && Y[rm] != f)
          hrec[atomicAdd(&ch[rm - 1], 1)] = pack_ix(f, min(a.x, b.x) - c.ox, max(a.x, b.x) - c.ox);
      }
    }
  }
  return base;
}

// The culled lists of region R = [X0, X1) x [Y0, Y1), region (rx, ry) of the
// pair's nx x ny split, from polygon s's index at blk (see build_index):
// the same sets as build_local(R), corner parity from the header.
__device__ bool cull_index(const uint64_t* blk, int nx, int ny, int rx, int ry, int X0, int Y0, int X1, int Y1,
                           LocalPoly& L) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const int Wr = X1 - X0, Hr = Y1 - Y0;
  const unsigned* hdr = reinterpret_cast<const unsigned*>(blk);
  const int vs = (int)hdr[rx], ve = (int)hdr[rx + 1], totv = (int)hdr[nx];
  const int hs = (int)hdr[nx + 1 + ry], he = (int)hdr[nx + 1 + ry + 1];
  L.pi = (int)((hdr[nx + ny + 2 + ry] >> rx) & 1u);
  const uint64_t* vrec = blk + ix_header_words(nx, ny);
  const uint64_t* hrec = vrec + totv;
  int cnt = 0;
  for (int j0 = vs; j0 < ve; j0 += 32) {  // warp-uniform
    const int j = j0 + lane;
    bool keep = false;
    uint64_t rec = 0;
    if (j < ve) {
      int x, yl, yh;
      unpack_ix(vrec[j], x, yl, yh);  // x strictly inside the region's columns (its bucket)
      keep = yl < Y1 && yh > Y0;
      rec = pack_loc(x - X0, max(yl - Y0, -1), min(yh - Y0, Hr + 1));
    }
    const unsigned b = __ballot_sync(FULL, keep);
    const int pos = cnt + __popc(b & lt);
    if (keep && pos < kLCap) L.V[pos] = rec;
    cnt += __popc(b);
  }
  L.nV = cnt;
  cnt = 0;
  for (int j0 = hs; j0 < he; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    uint64_t rec = 0;
    if (j < he) {
      int f, xl, xh;
      unpack_ix(hrec[j], f, xl, xh);  // f strictly inside the region's rows
      keep = xl < X1 && xh > X0;
      rec = pack_loc(f - Y0, max(xl - X0, -1), min(xh - X0, Wr + 1));
    }
    const unsigned b = __ballot_sync(FULL, keep);
    const int pos = cnt + __popc(b & lt);
    if (keep && pos < kLCap) L.H[pos] = rec;
    cnt += __popc(b);
  }
  L.nH = cnt;
  return L.nV <= kLCap && L.nH <= kLCap;
}

// Lemma 1 (reading R6-A) for the sub-boxes of box B = [x0, x1) x [y0, y1)
// (region coords), edge-parallel over the local lists.  pi = parity of B's
// corner pixel (x0, y0).  hov: sub-boxes whose open interior meets an edge;
// par: parity of each sub-box's corner pixel = pi + crossings up B's left
// column (horizontal edges) + crossings along the sub-box's bottom row
// (vertical edges) -- all local.
__device__ __forceinline__ void classify_local(const LocalPoly& L, int x0, int y0, int Wb, int Hb, const Split& g,
                                               int pi, unsigned& hov, unsigned& par) {
  const int lane = threadIdx.x & 31;
  const int sx = 1 << g.lsx, sy = 1 << g.lsy;
  const unsigned kxmask = low_bits(g.kx);
  unsigned h = 0, p = 0;
  for (int j = lane; j < L.nV; j += 32) {
    int x, yl, yh;
    unpack_loc(L.V[j], x, yl, yh);
    x -= x0;
    yl -= y0;
    yh -= y0;
    if (yl < Hb && yh > 0) {
      const int r_hi = min(g.nrows - 1, (yh - 1) >> g.lsy);
      if (x > 0 && x < Wb && (x & (sx - 1)) != 0)  // edge inside a column's open x-range
        h |= (g.colpat << (x >> g.lsx)) & row_range(max(0, yl >> g.lsy), r_hi, g);
      if (x > 0) {  // crossed by the bottom row of sub-boxes (c, r) with c*sx >= x, yl <= r*sy < yh
        const int c_lo = (x + sx - 1) >> g.lsx;
        if (c_lo < g.ncols)
          p ^= ((kxmask & ~low_bits(c_lo)) * g.colpat) & row_range(max(0, (yl + sy - 1) >> g.lsy), r_hi, g);
      }
    }
  }
  for (int j = lane; j < L.nH; j += 32) {
    int y, xl, xh;
    unpack_loc(L.H[j], y, xl, xh);
    y -= y0;
    xl -= x0;
    xh -= x0;
    if (y > 0 && y < Hb && (y & (sy - 1)) != 0 && xl < Wb && xh > 0) {
      const int c_lo = max(0, xl >> g.lsx), c_hi = min(g.ncols - 1, (xh - 1) >> g.lsx);
      h |= low_bits(c_hi - c_lo + 1) << (((y >> g.lsy) << g.lkx) + c_lo);
    }
    if (xl <= 0 && xh > 0 && y > 0) {  // crosses B's left column above its corner: rows r with r*sy >= y
      const int r_lo = (y + sy - 1) >> g.lsy;
      if (r_lo < g.nrows) p ^= row_range(r_lo, g.nrows - 1, g);
    }
  }
  hov = __reduce_or_sync(FULL, h);
  par = __reduce_xor_sync(FULL, p) ^ (pi ? FULL : 0u);
}

// Pixelization of box B (region coords) for one polygon into staged buffers:
// vertical edges strictly inside B's columns crossing B's rows as
// {ylo, span, x, 0} (box-relative), horizontal edges crossing B's left column
// strictly inside B's rows as their row.  Returns counts (> kLStage: use the
// local lists directly).
__device__ __forceinline__ void stage_local(const LocalPoly& L, int x0, int y0, int x1, int y1, int4* sv, int* sh,
                                            int& nv, int& nh) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  int cnt = 0;
  for (int j0 = 0; j0 < L.nV; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    int x = 0, yl = 0, yh = 0;
    if (j < L.nV) {
      unpack_loc(L.V[j], x, yl, yh);
      keep = x > x0 && x < x1 && yl < y1 && yh > y0;
    }
    const unsigned b = __ballot_sync(FULL, keep);
    const int pos = cnt + __popc(b & lt);
    if (keep && pos < kLStage) sv[pos] = make_int4(yl - y0, yh - yl, x - x0, 0);
    cnt += __popc(b);
  }
  nv = cnt;
  cnt = 0;
  for (int j0 = 0; j0 < L.nH; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    int y = 0, xl = 0, xh = 0;
    if (j < L.nH) {
      unpack_loc(L.H[j], y, xl, xh);
      keep = xl <= x0 && xh > x0 && y > y0 && y < y1;
    }
    const unsigned b = __ballot_sync(FULL, keep);
    const int pos = cnt + __popc(b & lt);
    if (keep && pos < kLStage) sh[pos] = y - y0;
    cnt += __popc(b);
  }
  nh = cnt;
}

// Row word (row, columns xs .. xs+31 of box B) of one polygon: parity of the
// row's left-column pixel (pi + horizontal crossings), then one suffix mask
// per vertical edge inside B crossing the row (reading R19).
__device__ __forceinline__ unsigned row_word_local(const LocalPoly& L, const int4* sv, const int* sh, int nv, int nh,
                                                   int x0, int y0, int x1, int y1, int pi, int row, int xs) {
  int par = pi;
  unsigned m = 0;
  if (nh <= kLStage) {
    for (int t = 0; t < nh; t++) par ^= (sh[t] <= row) ? 1 : 0;
  } else {
    for (int t = 0; t < L.nH; t++) {
      int y, xl, xh;
      unpack_loc(L.H[t], y, xl, xh);
      par ^= (xl <= x0 && xh > x0 && y > y0 && y < y1 && y - y0 <= row) ? 1 : 0;
    }
  }
  if (nv <= kLStage) {
#pragma unroll 4
    for (int t = 0; t < nv; t++) {
      const int4 r = sv[t];
      if ((unsigned)(row - r.x) < (unsigned)r.y) m ^= suffix_mask(r.z - xs);
    }
  } else {
    for (int t = 0; t < L.nV; t++) {
      int x, yl, yh;
      unpack_loc(L.V[t], x, yl, yh);
      if (x > x0 && x < x1 && (unsigned)(row + y0 - yl) < (unsigned)(yh - yl)) m ^= suffix_mask(x - x0 - xs);
    }
  }
  return m ^ (par ? FULL : 0u);
}

// Pixelization of a small box B (region coords) by crossing parity, one
// (row, 32-column word) per lane: (|B n p n q|, |B n (p u q)|); the union only
// when `uni` (modes 1 and 2 count it directly).
template <bool COUNT>
__device__ longlong2 pixelize_rows(const LocalPoly& P, const LocalPoly& Q, int x0, int y0, int x1, int y1, int pip,
                                    int piq, bool uni, int4* sv, int* sh, long long* counters) {
  const int lane = threadIdx.x & 31;
  int nvp, nhp, nvq, nhq;
  stage_local(P, x0, y0, x1, y1, sv, sh, nvp, nhp);
  stage_local(Q, x0, y0, x1, y1, sv + kLStage, sh + kLStage, nvq, nhq);
  __syncwarp();
  const int Wb = x1 - x0, Hb = y1 - y0, nw = (Wb + 31) >> 5, nseg = Hb * nw;
  long long ai = 0, au = 0;
  for (int s0 = 0; s0 < nseg; s0 += 32) {
    const int s = s0 + lane;
    if (s < nseg) {
      const int row = s / nw, xs = (s - row * nw) << 5;
      const unsigned mp = row_word_local(P, sv, sh, nvp, nhp, x0, y0, x1, y1, pip, row, xs);
      const unsigned mq = row_word_local(Q, sv + kLStage, sh + kLStage, nvq, nhq, x0, y0, x1, y1, piq, row, xs);
      const unsigned valid = low_bits(Wb - xs);
      ai += __popc(mp & mq & valid);
      if (uni) au += __popc((mp | mq) & valid);
    }
  }
  __syncwarp();
  if (COUNT && lane == 0) {
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXELS], (unsigned long long)Wb * Hb);
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROWTESTS], (unsigned long long)nseg * (nvp + nvq + nhp + nhq));
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXBOXES], 1ull);
  }
  return make_longlong2(ai, au);
}

// Pixelization of a larger box B (region coords), same results as
// pixelize_rows, row by row with the difference trick (the one prep uses for rasters): pixel
// (x, y) and pixel (x, y - 1) differ in inside-ness exactly when a horizontal
// edge on the line y spans column x, so row y's words are row y - 1's XOR the
// range masks of the horizontal edges at y.  Only the box's first row is found
// by crossing parity (corner parity + one suffix mask per vertical edge, R19);
// every further row costs its share of the horizontal edges plus a prefix XOR.
// The box is processed in column strips of <= 128 pixels (4 words) and bands
// of rows that fit the row buffer (the staging area, reused once the first row
// is done); a band starts from the previous band's last row.
constexpr int kDWords = (int)((2 * kLStage * sizeof(int4) + 2 * kLStage * sizeof(int)) / sizeof(unsigned) / 2);

template <bool COUNT>
__device__ longlong2 pixelize_bands(const LocalPoly& P, const LocalPoly& Q, int x0, int y0, int x1, int y1, int pip,
                                    int piq, bool uni, int4* sv, int* sh, long long* counters) {
  const int lane = threadIdx.x & 31;
  unsigned* DP = reinterpret_cast<unsigned*>(sv);  // row words, [row][word], per polygon
  unsigned* DQ = DP + kDWords;
  const int Wb = x1 - x0, Hb = y1 - y0;
  long long ai = 0, au = 0;
  unsigned long long tests = 0;
  for (int sx = 0; sx < Wb; sx += 128) {  // column strips (warp-uniform)
    const int sw = min(128, Wb - sx), nw = (sw + 31) >> 5;
    const int RB = kDWords / nw;
    // first row of the strip by crossing parity: lanes 0..nw-1 for p, 8..8+nw-1 for q
    int nvp, nhp, nvq, nhq;
    stage_local(P, x0, y0, x1, y1, sv, sh, nvp, nhp);
    stage_local(Q, x0, y0, x1, y1, sv + kLStage, sh + kLStage, nvq, nhq);
    __syncwarp();
    unsigned carry = 0;
    if (lane < nw)
      carry = row_word_local(P, sv, sh, nvp, nhp, x0, y0, x1, y1, pip, 0, sx + 32 * lane);
    else if (lane >= 8 && lane < 8 + nw)
      carry = row_word_local(Q, sv + kLStage, sh + kLStage, nvq, nhq, x0, y0, x1, y1, piq, 0, sx + 32 * (lane - 8));
    if (COUNT) tests += (unsigned long long)nw * (nvp + nvq);
    __syncwarp();  // the staging area becomes the row buffer
    for (int by = 0; by < Hb; by += RB) {  // bands of rows (warp-uniform)
      const int rb = min(RB, Hb - by);
      for (int i = lane; i < rb * nw; i += 32) DP[i] = DQ[i] = 0u;
      __syncwarp();
      if (lane < nw) DP[lane] = carry;  // band row 0 starts from the row below it
      if (lane >= 8 && lane < 8 + nw) DQ[lane - 8] = carry;
      __syncwarp();
      // horizontal edges on the lines y0 + by + r (r >= 1 in the first band):
      // toggle row r over the strip columns they span
      const int cx0 = x0 + sx, cx1 = x0 + sx + sw;
      for (int side = 0; side < 2; side++) {
        const LocalPoly& L = side ? Q : P;
        unsigned* D = side ? DQ : DP;
        for (int t = lane; t < L.nH; t += 32) {
          int y, xl, xh;
          unpack_loc(L.H[t], y, xl, xh);
          const int r = y - y0 - by;
          const int a = max(xl, cx0) - cx0, b = min(xh, cx1) - cx0;
          if (y > y0 && r >= 0 && r < rb && a < b)
            for (int w = a >> 5; w <= (b - 1) >> 5; w++)
              atomicXor(&D[r * nw + w], low_bits(min(b - 32 * w, 32)) & ~low_bits(max(a - 32 * w, 0)));
        }
      }
      __syncwarp();
      // prefix XOR down the rows: four lanes per (polygon, word) sequence
      {
        const int g = lane >> 2, sub = lane & 3, w = g & 3;
        unsigned* D = (g >> 2) ? DQ : DP;
        const bool act = w < nw;
        const int per = (rb + 3) >> 2, r0 = min(rb, sub * per), r1 = min(rb, r0 + per);
        unsigned tot = 0;
        if (act)
          for (int r = r0; r < r1; r++) tot ^= D[r * nw + w];
        unsigned ex = tot;  // exclusive XOR-scan over the group's 4 lanes
        unsigned v = __shfl_up_sync(0xffffffffu, ex, 1, 4);
        ex = sub >= 1 ? ex ^ v : ex;
        v = __shfl_up_sync(0xffffffffu, ex, 2, 4);
        ex = sub >= 2 ? ex ^ v : ex;
        ex ^= tot;
        if (act) {
          unsigned acc = ex;
          for (int r = r0; r < r1; r++) {
            acc ^= D[r * nw + w];
            D[r * nw + w] = acc;
          }
        }
      }
      __syncwarp();
      // word index i % nw, kept incrementally (no integer modulo in the loop)
      for (int i = lane, w = lane % nw, step = 32 % nw; i < rb * nw; i += 32, w = w + step >= nw ? w + step - nw : w + step) {
        const unsigned valid = low_bits(sw - 32 * w);
        const unsigned mp = DP[i], mq = DQ[i];
        ai += __popc(mp & mq & valid);
        if (uni) au += __popc((mp | mq) & valid);
      }
      if (lane < nw) carry = DP[(rb - 1) * nw + lane];
      if (lane >= 8 && lane < 8 + nw) carry = DQ[(rb - 1) * nw + lane - 8];
      __syncwarp();
    }
  }
  if (COUNT) {
    if (lane == 0) {  // tests is warp-uniform
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXELS], (unsigned long long)Wb * Hb);
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROWTESTS], tests);
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXBOXES], 1ull);
    }
  }
  return make_longlong2(ai, au);
}

// Boxes of up to eight (row, word) items per lane pixelize by crossing parity;
// larger ones by bands (first row by crossings, the rest by the difference
// trick), whose cost grows with edges + rows instead of edges x rows.
template <bool COUNT>
__device__ __forceinline__ longlong2 pixelize_local(const LocalPoly& P, const LocalPoly& Q, int x0, int y0, int x1,
                                                   int y1, int pip, int piq, bool uni, int4* sv, int* sh,
                                                   long long* counters) {
  if ((y1 - y0) * ((x1 - x0 + 31) >> 5) <= 256)
    return pixelize_rows<COUNT>(P, Q, x0, y0, x1, y1, pip, piq, uni, sv, sh, counters);
  return pixelize_bands<COUNT>(P, Q, x0, y0, x1, y1, pip, piq, uni, sv, sh, counters);
}

// sampling-box stack entry: x0, y0, x1, y1 (15 bit each, region coords), parity bits of both polygons
__device__ __forceinline__ uint64_t pack_sb(int x0, int y0, int x1, int y1, int pp, int pq) {
  return (uint64_t)x0 | ((uint64_t)y0 << 15) | ((uint64_t)x1 << 30) | ((uint64_t)y1 << 45) | ((uint64_t)pp << 60) |
         ((uint64_t)pq << 61);
}

// Algorithm 1 on one region with local lists (DFS, warp-private stack).
// mode 0 = PixelBox (intersection only; the union follows from the areas),
// mode 1 = PixelOnly (pixelize the region, count both), mode 2 = PixelBox-NoSep
// (§5.2: a box is decided only when both its intersection and union
// contributions are).  Returns this lane's (I, U) share.
template <bool COUNT>
__device__ longlong2 region_pixelbox(const LocalPoly& P, const LocalPoly& Q, int Wr, int Hr, int T, int mode, int dense,
                                     uint64_t* stk, int4* sv, int* sh, long long* counters, unsigned& status) {
  const int lane = threadIdx.x & 31;
  const bool uni = mode != 0;
  if (mode == 1 || (long long)Wr * Hr < T)
    return pixelize_local<COUNT>(P, Q, 0, 0, Wr, Hr, P.pi, Q.pi, uni, sv, sh, counters);
  long long ai = 0, au = 0;
  if (lane == 0) stk[0] = pack_sb(0, 0, Wr, Hr, P.pi, Q.pi);
  int top = 1;
  __syncwarp();
  while (top > 0) {
    const uint64_t e = stk[top - 1];
    top--;
    __syncwarp();  // every lane has read the popped entry before it is overwritten (reading R11)
    const int x0 = (int)(e & 0x7fff), y0 = (int)((e >> 15) & 0x7fff);
    const int x1 = (int)((e >> 30) & 0x7fff), y1 = (int)((e >> 45) & 0x7fff);
    const int pip = (int)((e >> 60) & 1), piq = (int)((e >> 61) & 1);
    const int Wb = x1 - x0, Hb = y1 - y0;
    if ((long long)Wb * Hb < T) {
      const longlong2 r = pixelize_local<COUNT>(P, Q, x0, y0, x1, y1, pip, piq, uni, sv, sh, counters);
      ai += r.x;
      au += r.y;
      continue;
    }
    const Split g = make_split(Wb, Hb);
    unsigned hp, pp, hq, pq;
    classify_local(P, x0, y0, Wb, Hb, g, pip, hp, pp);
    classify_local(Q, x0, y0, Wb, Hb, g, piq, hq, pq);
    const int cc = lane & (g.kx - 1), rr = lane >> g.lkx;
    const unsigned valid = __ballot_sync(FULL, cc < g.ncols && rr < g.nrows);
    const unsigned in_p = ~hp & pp, out_p = ~hp & ~pp, in_q = ~hq & pq, out_q = ~hq & ~pq;
    // BOXCONTRIBUTE / BOXCONTINUE (Alg. 1 l.33-35, reading R7)
    const unsigned i_dec = out_p | out_q | (in_p & in_q);
    const unsigned u_dec = in_p | in_q | (out_p & out_q);
    const unsigned cont = valid & ~(mode == 2 ? (i_dec & u_dec) : i_dec);
    const unsigned contrib_i = valid & in_p & in_q & ~cont;
    const unsigned contrib_u = valid & (in_p | in_q) & ~cont;
    const int ncont = __popc(cont);
    // Dense split: every sub-box is below T and most of them hover, so the next
    // level would stage edges for up to 32 small boxes; pixelizing B as one box
    // (bands: first row by crossings, then the difference trick) gives the same
    // exact count for less (an implementation choice, not Alg. 1's order; the
    // areas are identical by construction).
    if (SCCG_DENSE_SPLIT && dense && mode == 0 && ((long long)1 << (g.lsx + g.lsy)) < T &&
        ncont * SCCG_DENSE_DEN > __popc(valid) * SCCG_DENSE_NUM) {
      const longlong2 r = pixelize_local<COUNT>(P, Q, x0, y0, x1, y1, pip, piq, uni, sv, sh, counters);
      ai += r.x;
      au += r.y;
      continue;
    }
    const int sx0 = cc << g.lsx, sy0 = rr << g.lsy;
    const int sx1 = min(sx0 + (1 << g.lsx), Wb), sy1 = min(sy0 + (1 << g.lsy), Hb);
    const long long sz = (long long)(sx1 - sx0) * (sy1 - sy0);
    if ((contrib_i >> lane) & 1u) ai += sz;
    if (uni && ((contrib_u >> lane) & 1u)) au += sz;
    if (COUNT && lane == 0) {
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_BOXES], (unsigned long long)__popc(valid));
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_BOXEDGES], (unsigned long long)(P.nV + P.nH + Q.nV + Q.nH));
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_SPLITS], 1ull);
    }
    if (top + ncont > kLStack) {  // cannot happen for regions <= 32766 (depth <= 8 levels x 32); guard anyway
      status |= SCCG_STATUS_STACK;
      break;
    }
    if ((cont >> lane) & 1u)
      stk[top + __popc(cont & lanemask_lt())] =
          pack_sb(x0 + sx0, y0 + sy0, x0 + sx1, y0 + sy1, (int)((pp >> lane) & 1u), (int)((pq >> lane) & 1u));
    top += ncont;
    __syncwarp();
  }
  return make_longlong2(ai, au);
}

// ------------------------------------------------------------------ kernels
// mode 0: MBR(p) n MBR(q) (reading R5); modes 1, 2 count the union directly
// over the bounding box of MBR(p) u MBR(q).
__device__ __forceinline__ int4 root_box(const DevSet& Ps, const DevSet& Qs, int2 pq, int mode) {
  const int4 mp = Ps.mbr[pq.x], mq = Qs.mbr[pq.y];
  if (mode != 0) return make_int4(min(mp.x, mq.x), min(mp.y, mq.y), max(mp.z, mq.z), max(mp.w, mq.w));
  return make_int4(max(mp.x, mq.x), max(mp.y, mq.y), min(mp.z, mq.z), min(mp.w, mq.w));
}

constexpr size_t kLSmemPerWarp = (size_t)4 * kLCap * sizeof(uint64_t) + (size_t)2 * kLStage * sizeof(int4) +
                                 (size_t)2 * kLStage * sizeof(int) + (size_t)kLStack * sizeof(uint64_t) +
                                 (size_t)kLItems * sizeof(int4);
constexpr size_t kLSmem = kLWarps * kLSmemPerWarp;

template <bool COUNT>
#ifndef SCCG_ITEM_MINB
#define SCCG_ITEM_MINB 4  // item-kernel CTAs per SM (registers: 4 -> up to 128 per thread)
#endif
__global__ void __launch_bounds__(kLWarps * 32, SCCG_ITEM_MINB)
    item_kernel(DevSet Ps, DevSet Qs, const int2* __restrict__ pairs, LargeWs w, int T, int mode, int dense,
                long long* __restrict__ inter, long long* __restrict__ uni, long long* counters, sccg_sums* sums,
                unsigned* __restrict__ hit_p, unsigned* __restrict__ hit_q) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_entry();  // the small kernel's items and counters
  unsigned char* base = s_raw + (size_t)warp * kLSmemPerWarp;
  LocalPoly P, Q;
  P.V = reinterpret_cast<uint64_t*>(base);
  P.H = P.V + kLCap;
  Q.V = P.H + kLCap;
  Q.H = Q.V + kLCap;
  int4* sv = reinterpret_cast<int4*>(Q.H + kLCap);
  int* sh = reinterpret_cast<int*>(sv + 2 * kLStage);
  uint64_t* stk = reinterpret_cast<uint64_t*>(sh + 2 * kLStage);
  int4* istk = reinterpret_cast<int4*>(stk + kLStack);
  const long long n_cap = w.n_cap;
  const long long nl = min((long long)(ld_coherent(reinterpret_cast<const long long*>(w.ctr) + 2) & 0xffffffffll), n_cap);
  const long long ne = min(ld_coherent(reinterpret_cast<const long long*>(w.ctr) + 1), w.extra_cap);
  const long long total = nl + ne;
  if (total == 0) return;  // no large pairs in this batch
  unsigned status = 0;
  // batch totals of the pairs this warp finalizes (lane 0)
  unsigned long long a_n = 0, a_nz = 0, a_i = 0, a_u = 0, a_ap = 0, a_aq = 0, l0 = 0, l1 = 0, l2 = 0, l3 = 0, rootpx = 0;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(&w.ctr[0], 1ull);
    t = __shfl_sync(FULL, t, 0);
    if ((long long)t >= total) break;
    const uint64_t it = w.items[(long long)t < nl ? (long long)t : n_cap + ((long long)t - nl)];
    const unsigned i = (unsigned)(it & 0xffffffffu);
    if (i == 0xffffffffu) continue;
    const int rx = (int)((it >> 32) & 0xff), ry = (int)((it >> 40) & 0xff);
    const int nx = (int)((it >> 48) & 0xff), ny = (int)((it >> 56) & 0xff);
    const long long k = w.list[i];
    const int2 pq = pairs[k];
    const int4 rb = root_box(Ps, Qs, pq, mode);
    const int W = rb.z - rb.x, H = rb.w - rb.y;
    PolyRef pr[2];
    for (int s = 0; s < 2; s++) {
      const DevSet& S = s ? Qs : Ps;
      const int id = s ? pq.y : pq.x;
      const int4 m = S.mbr[id];
      const long long o = S.off[id];
      pr[s].ev = S.edges + o;
      pr[s].v = S.xy + o;
      const int2 ec = S.ecount[id];
      pr[s].nv = ec.x & kNvMask;
      pr[s].o0 = (unsigned)ec.y;
      pr[s].V = (int)(S.off[id + 1] - o);
      pr[s].dx = m.x - rb.x;
      pr[s].dy = m.y - rb.y;
      pr[s].ox = rb.x;
      pr[s].oy = rb.y;
    }
    long long acc = 0, acc_u = 0;
    // the pair's edge index: built by the warp holding its first item, used
    // by the others once ready (else they cull directly)
    long long ixb = -1;
    // only worth it when the first items alone keep every warp busy for a few
    // rounds, so the extra items (queued after all first items) find their
    // index built instead of racing the build
    if (w.pool && nx * ny >= kIxMin && nl >= 4ll * gridDim.x * kLWarps) {
      if ((long long)t < nl) {
        ixb = build_index(pr, W, H, nx, ny, w, reinterpret_cast<int*>(sv));
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          if (ixb >= 0) w.ixoff[i] = ixb;
          __threadfence();
          st_release_i(&w.ixstate[i], ixb >= 0 ? kIxReady : kIxNone);
        }
      } else if (ld_acquire_i(&w.ixstate[i]) == kIxReady) {
        ixb = w.ixoff[i];
      }
    }
    // in-warp item stack: the region, split in two while its local lists overflow
    if (lane == 0)
      istk[0] = make_int4((int)((long long)rx * W / nx), (int)((long long)ry * H / ny),
                          (int)((long long)(rx + 1) * W / nx), (int)((long long)(ry + 1) * H / ny));
    int itop = 1;
    bool whole = true;  // the popped region is the item's own region (not a split of it)
    __syncwarp();
    while (itop > 0) {
      const int4 R = istk[itop - 1];
      itop--;
      __syncwarp();
      const int Wr = R.z - R.x, Hr = R.w - R.y;
      bool fits = Wr <= kMaxRegion && Hr <= kMaxRegion;
      if (fits && whole && ixb >= 0) {
        const uint64_t* b0 = w.pool + ixb;
        const unsigned* h0 = reinterpret_cast<const unsigned*>(b0);
        const uint64_t* b1 = b0 + ix_header_words(nx, ny) + h0[nx] + h0[nx + 1 + ny];
        const bool a = cull_index(b0, nx, ny, rx, ry, R.x, R.y, R.z, R.w, P);
        const bool b = cull_index(b1, nx, ny, rx, ry, R.x, R.y, R.z, R.w, Q);
        fits = a && b;
      } else if (fits) {
        const bool a = build_local(pr[0], R.x, R.y, R.z, R.w, P);
        const bool b = build_local(pr[1], R.x, R.y, R.z, R.w, Q);
        fits = a && b;
      }
      whole = false;
      __syncwarp();
      if (!fits) {
        if (itop + 2 > kLItems) {
          status |= SCCG_STATUS_STACK;
          continue;
        }
        if (lane == 0) {
          if (Wr >= Hr) {
            const int xm = R.x + Wr / 2;
            istk[itop] = make_int4(R.x, R.y, xm, R.w);
            istk[itop + 1] = make_int4(xm, R.y, R.z, R.w);
          } else {
            const int ym = R.y + Hr / 2;
            istk[itop] = make_int4(R.x, R.y, R.z, ym);
            istk[itop + 1] = make_int4(R.x, ym, R.z, R.w);
          }
        }
        itop += 2;
        __syncwarp();
        continue;
      }
      const longlong2 r = region_pixelbox<COUNT>(P, Q, Wr, Hr, T, mode, dense, stk, sv, sh, counters, status);
      acc += r.x;
      acc_u += r.y;
      __syncwarp();
    }
    acc = (long long)warp_sum_u64((unsigned long long)acc);
    if (mode != 0) acc_u = (long long)warp_sum_u64((unsigned long long)acc_u);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&w.acc[i]), (unsigned long long)acc);
      if (mode != 0) atomicAdd(reinterpret_cast<unsigned long long*>(&w.acc_u[i]), (unsigned long long)acc_u);
      __threadfence();
      if (atomicSub(&w.rem[i], 1u) == 1u) {  // last region of the pair: finalize it
        __threadfence();
        const long long I = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&w.acc[i]), 0ull);
        const long long ap = Ps.area[pq.x], aq = Qs.area[pq.y];
        // indirect union; counted directly by the §5.2 baselines
        const long long U = mode == 0 ? ap + aq - I
                                      : (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&w.acc_u[i]), 0ull);
        if (inter) inter[k] = I;
        if (uni) uni[k] = U;
        a_n++;
        a_i += I;
        a_ap += ap;
        a_aq += aq;
        if (I != 0) {
          if (hit_p) atomicOr(&hit_p[pq.x >> 5], 1u << (pq.x & 31));
          if (hit_q) atomicOr(&hit_q[pq.y >> 5], 1u << (pq.y & 31));
          unsigned long long b0, b1, b2, b3;
          ratio_limbs(I, U, b0, b1, b2, b3);
          a_nz++;
          a_u += U;
          l0 += b0;
          l1 += b1;
          l2 += b2;
          l3 += b3;
        }
        if (COUNT) rootpx += (unsigned long long)W * H;
      }
    }
  }
  status = __reduce_or_sync(FULL, status);
  if (lane == 0) {
    if (status) atomicOr(reinterpret_cast<unsigned long long*>(&sums->status), (unsigned long long)status);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(sums);
    const unsigned long long v[10] = {a_n, a_nz, a_i, a_u, a_ap, a_aq, l0, l1, l2, l3};
    for (int f = 0; f < 10; f++)
      if (v[f]) atomicAdd(d + f, v[f]);
    if (COUNT && rootpx) atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROOTPX], rootpx);
  }
}

// ---------------------------------------------------------------------- host
static long long extra_cap_for(long long n_cap) { return 4 * n_cap + 65536; }

static size_t large_layout(long long n_cap, Carve& cv, LargeWs& w) {
  const long long n = n_cap > 0 ? n_cap : 1;
  w.ctr = cv.take<unsigned long long>(4);
  w.list = cv.take<long long>(n);
  w.acc = cv.take<long long>(n);
  w.acc_u = cv.take<long long>(n);
  w.rem = cv.take<unsigned>(n);
  w.ixstate = cv.take<int>(n);
  w.ixoff = cv.take<long long>(n);
  w.n_cap = n_cap;
  w.extra_cap = extra_cap_for(n_cap);
  w.items = cv.take<uint64_t>(n + w.extra_cap);
  w.pool = nullptr;
  w.pool_cap = 0;
  return cv.used;
}

size_t large_ws_bytes(long long n_cap) {
  Carve cv{nullptr, ~size_t(0)};
  LargeWs w;
  return large_layout(n_cap, cv, w) + 256;
}

LargeWs large_ws(long long n_cap, void* ws, size_t ws_bytes, void* pool, size_t pool_bytes, bool& ok) {
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  LargeWs w;
  large_layout(n_cap, cv, w);
  ok = cv.ok && ws != nullptr;
  if (pool && pool_bytes >= 4096) {  // optional edge-index pool (8-byte words, 16-byte aligned by the caller)
    w.pool = reinterpret_cast<uint64_t*>(pool);
    w.pool_cap = (long long)(pool_bytes / 8);
  }
  return w;
}

int launch_large(const DevSet& Ps, const DevSet& Qs, const int2* pairs, const LargeWs& w, long long* inter,
                 long long* uni, sccg_sums* sums, int T, int mode, int dense, long long* counters, unsigned* hit_p,
                 unsigned* hit_q, cudaStream_t stream) {
  static cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(item_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(item_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLSmem);
    return e;
  }();
  if (int r = check_cuda(attr, "item kernel smem attribute")) return r;
  static int sms = 0, per_sm[2] = {0, 0};
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], item_kernel<false>, kLWarps * 32, kLSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], item_kernel<true>, kLWarps * 32, kLSmem);
  }
  const bool count = counters != nullptr;
  const unsigned ib = (unsigned)(sms * max(per_sm[count], 1));
  cudaError_t e;
  if (count)
    e = launch_pdl(item_kernel<true>, dim3(ib), dim3(kLWarps * 32), kLSmem, stream, Ps, Qs, pairs, w, T, mode, dense, inter,
                   uni, counters, sums, hit_p, hit_q);
  else
    e = launch_pdl(item_kernel<false>, dim3(ib), dim3(kLWarps * 32), kLSmem, stream, Ps, Qs, pairs, w, T, mode, dense, inter,
                   uni, (long long*)nullptr, sums, hit_p, hit_q);
  if (int r = check_cuda(e, "pixelbox large launch")) return r;
  return check_cuda(cudaGetLastError(), "pixelbox large launch");
}

}  // namespace sccg
