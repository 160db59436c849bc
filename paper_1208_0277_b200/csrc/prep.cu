// prep.cu -- per-polygon prep, one warp per polygon.
//
// For each ring: the half-open pixel MBR; the area by the shoelace formula
// A = 1/2 |sum_i (x_i y_{i+1} - x_{i+1} y_i)| with "different threads compute
// different vertices and sum up the partial results" (§3.2),
// evaluated on MBR-rebased coordinates in int64 (translation invariant, no
// overflow); validation (rectilinear edges, ranges, offsets); and the 8-byte
// edge records PixelBox streams (vertical edges compacted to the front of the
// polygon's vertex slot, horizontal edges to the back).
#include "internal.cuh"

namespace sccg {

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bit, int64_t poly) {
  atomicOr(&status[0], bit);
  atomicMin(&status[1], (uint32_t)min(poly, (int64_t)0x7fffffff));
}

__global__ void __launch_bounds__(256) prep_kernel(const int2* __restrict__ xy, const int64_t* __restrict__ off,
                                                   int64_t n, int64_t nv_total, int4* __restrict__ mbr,
                                                   int64_t* __restrict__ area, int2* __restrict__ ecount,
                                                   uint64_t* __restrict__ edges, uint32_t* __restrict__ status,
                                                   int validate) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t poly = warp; poly < n; poly += nwarps) {
    const int64_t b = off[poly], e = off[poly + 1];
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
    // pass 1: MBR
    int xmin = INT_MAX, ymin = INT_MAX, xmax = INT_MIN, ymax = INT_MIN;
    bool bad_range = false;
    for (int64_t i = lane; i < V; i += 32) {
      int2 v = xy[b + i];
      xmin = min(xmin, v.x);
      xmax = max(xmax, v.x);
      ymin = min(ymin, v.y);
      ymax = max(ymax, v.y);
      bad_range |= (int64_t)v.x > kMaxCoord || (int64_t)v.x < -kMaxCoord || (int64_t)v.y > kMaxCoord ||
                   (int64_t)v.y < -kMaxCoord;
    }
    xmin = __reduce_min_sync(0xffffffffu, xmin);
    ymin = __reduce_min_sync(0xffffffffu, ymin);
    xmax = __reduce_max_sync(0xffffffffu, xmax);
    ymax = __reduce_max_sync(0xffffffffu, ymax);
    bad_range = __any_sync(0xffffffffu, bad_range) || (int64_t)xmax - xmin > kMaxExtent ||
                (int64_t)ymax - ymin > kMaxExtent;
    // pass 2: shoelace terms, validation, edge records
    long long twice_area = 0;
    bool diag = false;
    int nvert = 0, nhor = 0;
    for (int64_t i0 = 0; i0 < V; i0 += 32) {
      const int64_t i = i0 + lane;
      bool is_v = false, is_h = false;
      uint64_t rec = 0;
      if (i < V) {
        int2 a = xy[b + i];
        int2 c = xy[b + (i + 1 == V ? 0 : i + 1)];
        long long ax = a.x - xmin, ay = a.y - ymin, cx = c.x - xmin, cy = c.y - ymin;
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
      unsigned bv = __ballot_sync(0xffffffffu, is_v), bh = __ballot_sync(0xffffffffu, is_h);
      if (!bad_range) {
        if (is_v) edges[b + nvert + __popc(bv & lanemask_lt())] = rec;
        if (is_h) edges[e - 1 - (nhor + __popc(bh & lanemask_lt()))] = rec;
      }
      nvert += __popc(bv);
      nhor += __popc(bh);
    }
    for (int o = 16; o; o >>= 1) twice_area += __shfl_xor_sync(0xffffffffu, twice_area, o);
    diag = __any_sync(0xffffffffu, diag);
    if (lane == 0) {
      long long a2 = twice_area < 0 ? -twice_area : twice_area;
      area[poly] = a2 / 2;
      mbr[poly] = make_int4(xmin, ymin, xmax, ymax);
      ecount[poly] = bad_range ? make_int2(0, 0) : make_int2(nvert, nhor);
      if (validate && diag) flag(status, SCCG_STATUS_NOT_RECTILINEAR, poly);
      if (bad_range) flag(status, SCCG_STATUS_RANGE, poly);
    }
  }
}

__global__ void status_init_kernel(uint32_t* status) {
  status[0] = 0;
  status[1] = 0xffffffffu;
}

cudaError_t launch_prep(const sccg_polyset* s, int validate, cudaStream_t st) {
  status_init_kernel<<<1, 1, 0, st>>>(s->status);
  if (s->n_polygons > 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t warps_needed = s->n_polygons;
    int64_t blocks = (warps_needed + 7) / 8;
    int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread blocks per SM
    if (blocks > cap) blocks = cap;
    prep_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const int2*>(s->xy), s->offsets, s->n_polygons,
                                                  s->n_vertices, reinterpret_cast<int4*>(s->mbr), s->area,
                                                  reinterpret_cast<int2*>(s->ecount), s->edges, s->status, validate);
  }
  return cudaGetLastError();
}

}  // namespace sccg
