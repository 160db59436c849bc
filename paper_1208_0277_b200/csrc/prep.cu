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
// HBM-bound pass: a CTA stages the vertex range of 64 consecutive polygons
// (one coalesced sweep) in shared memory, then each warp derives its polygons
// from shared memory.  Ranges larger than the tile fall back to reading the
// polygon's vertices from global memory (same code, other pointer).
#include "internal.cuh"

namespace sccg {

constexpr int kPrepThreads = 128;
constexpr int kPrepPolys = 128;   // one ring per thread per tile
constexpr int kPrepVerts = 5120;  // 40 KB of int2 staged per tile (dynamic shared memory)

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
                                             int validate) {
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
  if (lane == 0) {
    area[poly] = (twice_area < 0 ? -twice_area : twice_area) / 2;
    mbr[poly] = m;
    ecount[poly] = make_int2(nvert, nhor);
    if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
  }
  return m;
}

// One polygon by one thread (the common small ring): same results as
// prep_polygon, serial over the ring's vertices in the shared-memory tile,
// 32-bit arithmetic on MBR-rebased coordinates (extents <= 65535, so each
// shoelace product fits 32 bits unsigned; the sum is int64).  Records are
// written in place over the ring's own vertex slot: record k lands in slot
// k <= i - 1 while vertex i is being read.
__device__ __forceinline__ int4 prep_polygon_thread(int2* v, int V, int64_t poly, int4* __restrict__ mbr,
                                                    int64_t* __restrict__ area, int2* __restrict__ ecount,
                                                    uint32_t* __restrict__ status, int validate) {
  int xmin = INT_MAX, ymin = INT_MAX, xmax = INT_MIN, ymax = INT_MIN;
#pragma unroll 4
  for (int i = 0; i < V; i++) {
    const int2 a = v[i];
    xmin = min(xmin, a.x);
    xmax = max(xmax, a.x);
    ymin = min(ymin, a.y);
    ymax = max(ymax, a.y);
  }
  const int4 m = make_int4(xmin, ymin, xmax, ymax);
  mbr[poly] = m;
  if ((int64_t)xmin < -kMaxCoord || (int64_t)xmax > kMaxCoord || (int64_t)ymin < -kMaxCoord ||
      (int64_t)ymax > kMaxCoord || (int64_t)xmax - xmin > kMaxExtent || (int64_t)ymax - ymin > kMaxExtent) {
    area[poly] = 0;
    ecount[poly] = make_int2(0, 0);
    flag(status, SCCG_STATUS_RANGE, poly);
    return m;
  }
  uint64_t* out = reinterpret_cast<uint64_t*>(v);
  long long twice_area = 0;
  bool diag = false;
  int nvert = 0, nhor = 0;
  const unsigned fx = v[0].x - xmin, fy = v[0].y - ymin;
  unsigned ax = fx, ay = fy;
  auto edge = [&](unsigned cx, unsigned cy) {
    twice_area += (long long)(ax * cy) - (long long)(cx * ay);  // P:193, one term per vertex
    const bool is_v = ax == cx && ay != cy;
    nhor += (ay == cy && ax != cx) ? 1 : 0;
    diag |= ax != cx && ay != cy;
    const uint64_t rec = pack_edge(ax, min(ay, cy), max(ay, cy));
    if (is_v) out[nvert] = rec;
    nvert += is_v ? 1 : 0;
    ax = cx;
    ay = cy;
  };
  for (int i = 1; i < V; i++) {
    const int2 c = v[i];
    edge((unsigned)(c.x - xmin), (unsigned)(c.y - ymin));
  }
  edge(fx, fy);  // closing edge back to the first vertex
  area[poly] = (twice_area < 0 ? -twice_area : twice_area) / 2;
  // Raster: pixel (x, y) of the MBR is inside
  // iff an odd number of the row's vertical edges lie at or left of x (R19) --
  // PIXELINPOLY depends on the polygon alone, so it is computed once here.
  // Row r as a 32-bit word (bit x = column xlo + x): difference trick -- each
  // vertical edge XORs its suffix mask into rows lo and hi -- then a prefix XOR
  // over rows.  Stored in the slot's free tail (words 2 nv .. 2 nv + H), which
  // exists when 2 (V - nv) >= H; MBR width <= 32.
  const int W = xmax - xmin, H = ymax - ymin;
  bool raster = !diag && W <= 32 && 2 * (V - nvert) >= H;
  if (raster) {
    unsigned* D = reinterpret_cast<unsigned*>(out + nvert);
    for (int r = 0; r < H; r++) D[r] = 0u;
    for (int k = 0; k < nvert; k++) {
      int c, lo, hi;
      unpack_edge(out[k], c, lo, hi);
      const unsigned m = suffix_mask(c);
      D[lo] ^= m;
      if (hi < H) D[hi] ^= m;
    }
    unsigned acc = 0u;
    const unsigned wmask = low_bits(W);
    for (int r = 0; r < H; r++) {
      acc ^= D[r];
      D[r] = acc & wmask;
    }
  }
  ecount[poly] = make_int2(nvert, nhor | (raster ? kRasterFlag : 0));
  if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
  return m;
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

constexpr int kThreadMaxV = 192;  // rings up to this size are prepped by one thread

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const int2* __restrict__ xy,
                                                            const int64_t* __restrict__ off, int64_t n,
                                                            int64_t nv_total, int4* __restrict__ mbr,
                                                            int64_t* __restrict__ area, int2* __restrict__ ecount,
                                                            uint64_t* __restrict__ edges,
                                                            uint32_t* __restrict__ status, SetStats* stats,
                                                            int validate, int vec16) {
  extern __shared__ int4 s_dyn4[];  // kPrepVerts int2 (16-byte aligned)
  int2* s_xy = reinterpret_cast<int2*>(s_dyn4);
  __shared__ int64_t s_off[kPrepPolys + 1];
  __shared__ unsigned s_big[kPrepPolys / 32];
  __shared__ unsigned long long s_acc[4];
  __shared__ int s_b[6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StatAcc acc;
  acc.init();
  const int64_t ntiles = (n + kPrepPolys - 1) / kPrepPolys;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kPrepPolys;
    const int np = (int)min((int64_t)kPrepPolys, n - p0);
    __syncthreads();  // previous tile's shared data fully consumed
    for (int i = threadIdx.x; i <= np; i += blockDim.x) s_off[i] = off[p0 + i];
    if (threadIdx.x < kPrepPolys / 32) s_big[threadIdx.x] = 0;
    __syncthreads();
    // stage the tile's vertex range: 16-byte cp.async (LDGSTS) from an even
    // start, no register round trip, many copies in flight per thread
    const int64_t v0 = s_off[0] & ~int64_t(1), v1 = s_off[np];
    const bool tiled = s_off[0] >= 0 && v1 <= nv_total && v1 >= s_off[0] && v1 - v0 <= kPrepVerts;
    if (tiled) {
      const int64_t nv = v1 - v0;
      if (vec16) {
        const int64_t nvec = nv >> 1;
        const char* src = reinterpret_cast<const char*>(xy + v0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(s_dyn4);
        for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + (unsigned)(16 * i)), "l"(src + 16 * i));
        if ((nv & 1) && threadIdx.x == 0) s_xy[nv - 1] = xy[v1 - 1];
        asm volatile("cp.async.wait_all;\n" ::);
      } else {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) s_xy[i] = xy[v0 + i];
      }
    }
    __syncthreads();
    // thread per small ring (records in place in the tile)
    for (int j = threadIdx.x; j < np; j += blockDim.x) {
      const int64_t poly = p0 + j;
      const int64_t b = s_off[j], e = s_off[j + 1];
      const int64_t V = e - b;
      if (b < 0 || e > nv_total || V < 4) {  // malformed offsets or too few vertices
        mbr[poly] = make_int4(0, 0, 0, 0);
        area[poly] = 0;
        ecount[poly] = make_int2(0, 0);
        flag(status, SCCG_STATUS_ARG, poly);
        continue;
      }
      if (V > kThreadMaxV || !tiled) {
        atomicOr(&s_big[j >> 5], 1u << (j & 31));
        continue;
      }
      acc.add(prep_polygon_thread(s_xy + (b - v0), (int)V, poly, mbr, area, ecount, status, validate));
    }
    __syncthreads();
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
        const int4 m = prep_polygon(src, e - b, poly, out, mbr, area, ecount, status, validate);
        if (lane == 0) acc.add(m);
      }
    }
    __syncthreads();
    // coalesced write-out of the tile's records (16-byte stores when aligned)
    if (tiled) {
      const int64_t nv = v1 - v0;
      if (vec16 && (reinterpret_cast<uintptr_t>(edges) & 15) == 0) {
        int4* dst = reinterpret_cast<int4*>(edges + v0);
        for (int64_t i = threadIdx.x; i < (nv >> 1); i += blockDim.x) dst[i] = s_dyn4[i];
        if ((nv & 1) && threadIdx.x == 0) edges[v1 - 1] = reinterpret_cast<const uint64_t*>(s_xy)[nv - 1];
      } else {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) edges[v0 + i] = reinterpret_cast<const uint64_t*>(s_xy)[i];
      }
    }
  }
  // block reduction of the statistics, then one atomic per field
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
}

__global__ void prep_init_kernel(uint32_t* status, SetStats* st) {
  if (threadIdx.x == 0) {
    status[0] = 0;
    status[1] = 0xffffffffu;
    st->bounds[0] = st->bounds[1] = INT_MAX;
    st->bounds[2] = st->bounds[3] = INT_MIN;
    st->maxext[0] = st->maxext[1] = 0;
    st->nonempty = st->sw = st->sh = st->swh = 0;
  }
}

cudaError_t launch_prep(const sccg_polyset* s, int validate, cudaStream_t st) {
  SetStats* stats = reinterpret_cast<SetStats*>(s->stats);
  prep_init_kernel<<<1, 32, 0, st>>>(s->status, stats);
  if (s->n_polygons > 0) {
    static cudaError_t attr = cudaFuncSetAttribute(prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)(kPrepVerts * sizeof(int2)));
    if (attr != cudaSuccess) return attr;
    static int sms = 0, per_sm = 1;
    if (sms == 0) {  // launch geometry, queried once per process
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep_kernel, kPrepThreads, kPrepVerts * sizeof(int2));
    }
    const int64_t ntiles = (s->n_polygons + kPrepPolys - 1) / kPrepPolys;
    int64_t blocks = ntiles;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    prep_kernel<<<(unsigned)blocks, kPrepThreads, kPrepVerts * sizeof(int2), st>>>(
        reinterpret_cast<const int2*>(s->xy), s->offsets, s->n_polygons, s->n_vertices,
        reinterpret_cast<int4*>(s->mbr), s->area, reinterpret_cast<int2*>(s->ecount), s->edges, s->status, stats,
        validate, (reinterpret_cast<uintptr_t>(s->xy) & 15) == 0 ? 1 : 0);
  }
  return cudaGetLastError();
}

}  // namespace sccg
