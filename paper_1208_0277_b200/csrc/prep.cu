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

constexpr int kPrepThreads = 256;
constexpr int kPrepPolys = 64;
constexpr int kPrepVerts = 5888;  // 46 KB of int2 (static shared memory limit 48 KB)

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bit, int64_t poly) {
  atomicOr(&status[0], bit);
  atomicMin(&status[1], (uint32_t)min(poly, (int64_t)0x7fffffff));
}

// One polygon by one warp; `v` points at its first vertex (shared or global).
__device__ __forceinline__ void prep_polygon(const int2* v, int64_t V, int64_t poly, int64_t b, int64_t e,
                                             int4* __restrict__ mbr, int64_t* __restrict__ area,
                                             int2* __restrict__ ecount, uint64_t* __restrict__ edges,
                                             uint32_t* __restrict__ status, int validate, int4& out_mbr) {
  const int lane = threadIdx.x & 31;
  int xmin = INT_MAX, ymin = INT_MAX, xmax = INT_MIN, ymax = INT_MIN;
  bool bad_range = false;
  for (int64_t i = lane; i < V; i += 32) {
    const int2 a = v[i];
    xmin = min(xmin, a.x);
    xmax = max(xmax, a.x);
    ymin = min(ymin, a.y);
    ymax = max(ymax, a.y);
    bad_range |= (int64_t)a.x > kMaxCoord || (int64_t)a.x < -kMaxCoord || (int64_t)a.y > kMaxCoord ||
                 (int64_t)a.y < -kMaxCoord;
  }
  xmin = __reduce_min_sync(0xffffffffu, xmin);
  ymin = __reduce_min_sync(0xffffffffu, ymin);
  xmax = __reduce_max_sync(0xffffffffu, xmax);
  ymax = __reduce_max_sync(0xffffffffu, ymax);
  bad_range = __any_sync(0xffffffffu, bad_range) || (int64_t)xmax - xmin > kMaxExtent ||
              (int64_t)ymax - ymin > kMaxExtent;
  long long twice_area = 0;
  bool diag = false;
  int nvert = 0, nhor = 0;
  for (int64_t i0 = 0; i0 < V; i0 += 32) {
    const int64_t i = i0 + lane;
    bool is_v = false, is_h = false;
    uint64_t rec = 0;
    if (i < V) {
      const int2 a = v[i];
      const int2 c = v[i + 1 == V ? 0 : i + 1];
      const long long ax = a.x - xmin, ay = a.y - ymin, cx = c.x - xmin, cy = c.y - ymin;
      twice_area += ax * cy - cx * ay;  // P:193, one term per thread
      if (a.x == c.x && a.y != c.y) {
        is_v = true;
        rec = pack_edge((uint32_t)ax, (uint32_t)min(ay, cy), (uint32_t)max(ay, cy));
      } else if (a.y == c.y && a.x != c.x) {
        is_h = true;
        rec = pack_edge((uint32_t)ay, (uint32_t)min(ax, cx), (uint32_t)max(ax, cx));
      } else if (a.x != c.x && a.y != c.y) {
        diag = true;
      }
    }
    const unsigned bv = __ballot_sync(0xffffffffu, is_v), bh = __ballot_sync(0xffffffffu, is_h);
    if (!bad_range) {
      if (is_v) edges[b + nvert + __popc(bv & lanemask_lt())] = rec;
      if (is_h) edges[e - 1 - (nhor + __popc(bh & lanemask_lt()))] = rec;
    }
    nvert += __popc(bv);
    nhor += __popc(bh);
  }
  for (int o = 16; o; o >>= 1) twice_area += __shfl_xor_sync(0xffffffffu, twice_area, o);
  diag = __any_sync(0xffffffffu, diag);
  out_mbr = make_int4(xmin, ymin, xmax, ymax);
  if (lane == 0) {
    const long long a2 = twice_area < 0 ? -twice_area : twice_area;
    area[poly] = a2 / 2;
    mbr[poly] = out_mbr;
    ecount[poly] = bad_range ? make_int2(0, 0) : make_int2(nvert, nhor);
    if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
    if (bad_range) flag(status, SCCG_STATUS_RANGE, poly);
  }
}

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const int2* __restrict__ xy,
                                                            const int64_t* __restrict__ off, int64_t n,
                                                            int64_t nv_total, int4* __restrict__ mbr,
                                                            int64_t* __restrict__ area, int2* __restrict__ ecount,
                                                            uint64_t* __restrict__ edges,
                                                            uint32_t* __restrict__ status, SetStats* stats,
                                                            int validate) {
  __shared__ int2 s_xy[kPrepVerts];
  __shared__ int64_t s_off[kPrepPolys + 1];
  __shared__ unsigned long long s_ent[kStatNK + 1];
  __shared__ int s_b[6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-thread (lane 0 of each warp) statistics
  unsigned long long ent[kStatNK];
#pragma unroll
  for (int k = 0; k < kStatNK; k++) ent[k] = 0;
  unsigned long long nonempty = 0;
  int bx0 = INT_MAX, by0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN, mw = 0, mh = 0;
  const int64_t ntiles = (n + kPrepPolys - 1) / kPrepPolys;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kPrepPolys;
    const int np = (int)min((int64_t)kPrepPolys, n - p0);
    __syncthreads();  // previous tile's shared data fully consumed
    for (int i = threadIdx.x; i <= np; i += blockDim.x) s_off[i] = off[p0 + i];
    __syncthreads();
    const int64_t v0 = s_off[0], v1 = s_off[np];
    const bool tiled = v0 >= 0 && v1 <= nv_total && v1 >= v0 && v1 - v0 <= kPrepVerts;
    if (tiled)
      for (int64_t i = threadIdx.x; i < v1 - v0; i += blockDim.x) s_xy[i] = xy[v0 + i];
    __syncthreads();
    for (int j = warp; j < np; j += kPrepThreads / 32) {
      const int64_t poly = p0 + j;
      const int64_t b = s_off[j], e = s_off[j + 1];
      const int64_t V = e - b;
      if (b < 0 || e > nv_total || V < 4) {  // malformed offsets or too few vertices
        if (lane == 0) {
          mbr[poly] = make_int4(0, 0, 0, 0);
          area[poly] = 0;
          ecount[poly] = make_int2(0, 0);
          flag(status, SCCG_STATUS_ARG, poly);
        }
        continue;
      }
      const bool in_smem = tiled && b >= v0 && e <= v1;
      int4 m;
      prep_polygon(in_smem ? s_xy + (b - v0) : xy + b, V, poly, b, e, mbr, area, ecount, edges, status, validate, m);
      if (lane == 0 && m.x < m.z && m.y < m.w) {  // join statistics over non-empty MBRs
        nonempty++;
        bx0 = min(bx0, m.x);
        by0 = min(by0, m.y);
        bx1 = max(bx1, m.z);
        by1 = max(by1, m.w);
        mw = max(mw, m.z - m.x);
        mh = max(mh, m.w - m.y);
#pragma unroll
        for (int k = 0; k < kStatNK; k++) {
          const int kk = k + kStatK0;
          const unsigned cx = (unsigned)(((m.z - 1) >> kk) - (m.x >> kk) + 1);
          const unsigned cy = (unsigned)(((m.w - 1) >> kk) - (m.y >> kk) + 1);
          ent[k] += (unsigned long long)cx * cy;
        }
      }
    }
  }
  // block reduction of the statistics, then one atomic per field
  if (threadIdx.x < kStatNK + 1) s_ent[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s_b[0] = s_b[1] = INT_MAX;
    s_b[2] = s_b[3] = INT_MIN;
    s_b[4] = s_b[5] = 0;
  }
  __syncthreads();
  if (lane == 0) {
    for (int k = 0; k < kStatNK; k++)
      if (ent[k]) atomicAdd(&s_ent[k], ent[k]);
    if (nonempty) {
      atomicAdd(&s_ent[kStatNK], nonempty);
      atomicMin(&s_b[0], bx0);
      atomicMin(&s_b[1], by0);
      atomicMax(&s_b[2], bx1);
      atomicMax(&s_b[3], by1);
      atomicMax(&s_b[4], mw);
      atomicMax(&s_b[5], mh);
    }
  }
  __syncthreads();
  if (threadIdx.x < kStatNK && s_ent[threadIdx.x]) atomicAdd(&stats->entries[threadIdx.x], s_ent[threadIdx.x]);
  if (threadIdx.x == 0 && s_ent[kStatNK]) {
    atomicAdd(&stats->nonempty, s_ent[kStatNK]);
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
    st->nonempty = 0;
  }
  if (threadIdx.x < kStatNK) st->entries[threadIdx.x] = 0;
}

cudaError_t launch_prep(const sccg_polyset* s, int validate, cudaStream_t st) {
  SetStats* stats = reinterpret_cast<SetStats*>(s->stats);
  prep_init_kernel<<<1, 32, 0, st>>>(s->status, stats);
  if (s->n_polygons > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ntiles = (s->n_polygons + kPrepPolys - 1) / kPrepPolys;
    int64_t blocks = ntiles;
    const int64_t cap = (int64_t)sms * 4;  // 4 resident 256-thread CTAs per SM (48 KB smem each)
    if (blocks > cap) blocks = cap;
    prep_kernel<<<(unsigned)blocks, kPrepThreads, 0, st>>>(
        reinterpret_cast<const int2*>(s->xy), s->offsets, s->n_polygons, s->n_vertices,
        reinterpret_cast<int4*>(s->mbr), s->area, reinterpret_cast<int2*>(s->ecount), s->edges, s->status, stats,
        validate);
  }
  return cudaGetLastError();
}

}  // namespace sccg
