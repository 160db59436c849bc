// join.cu -- MBR-overlap join by a uniform grid hash.
//
// The paper's filter stage searches a Hilbert R-tree on one CPU thread
// (§4.1) to produce "an array of polygon pairs with intersecting
// MBRs"; the predicate is the `&&` MBR test of Fig. 1(b), here
// half-open (reading R4).  On the GPU a uniform grid of 2^k-pixel cells is
// cheaper: Q's MBRs are bucketed into every cell they cover, each P MBR probes
// its cells, and a pair is emitted only from the cell holding its reference
// point (max xlo, max ylo) so it is found exactly once.  Each P's pairs are
// written to its own segment (exclusive scan of per-P counts) and sorted by q
// in place, so the output is sorted by (p, q) without a global sort.
//
// The cell size is chosen on the device from the per-set statistics sccg_prep
// gathered (no host round trip); the only host synchronisation is the final
// pair count the ABI returns.
#include <cub/device/device_scan.cuh>

#include "internal.cuh"

namespace sccg {

struct Grid {
  int k, cx0, cy0, ncx, ncy, empty;
  __device__ __forceinline__ int cell(int x, int y) const { return ((y >> k) - cy0) * ncx + ((x >> k) - cx0); }
};

__device__ __forceinline__ bool mbr_empty(const int4& m) { return m.x >= m.z || m.y >= m.w; }

static int64_t cell_cap(int64_t np, int64_t nq) { return np + nq + 1024; }
static int64_t entry_cap(int64_t nq) { return 8 * nq + 1024; }

// Upper bound and expectation of the 2^k-cell entries of one set (SetStats).
__device__ __forceinline__ void set_entries(const SetStats* s, int k, double& bound, double& expect) {
  const double c = 1.0 / (double)(1ll << k), n = (double)s->nonempty;
  const double sw = (double)s->sw, sh = (double)s->sh, swh = (double)s->swh;
  const double cont = swh * c * c + 2.0 * (sw + sh) * c + 4.0 * n;
  const double ext = n * (double)(((s->maxext[0] - 1) >> k) + 2) * (double)(((s->maxext[1] - 1) >> k) + 2);
  bound = cont < ext ? cont : ext;
  expect = n + (sw + sh) * c + swh * c * c;
}

// Cell size 2^k minimising the expected work E_p + E_q + C/4 + E_p E_q / C
// (bucket inserts + probes + scan + candidate tests) subject to the workspace
// caps on cells C and (upper-bounded) Q-entries.  Always feasible: once 2^k
// exceeds the largest MBR extent each MBR covers at most 2 x 2 cells.
__global__ void grid_select_kernel(const SetStats* __restrict__ sp, const SetStats* __restrict__ sq, long long ccap,
                                   long long ecap, Grid* g) {
  // one warp: lane j evaluates k = 3 + j (k <= 30), then an argmin over lanes
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  const bool empty = sp->nonempty == 0 || sq->nonempty == 0;
  const int xmin = min(sp->bounds[0], sq->bounds[0]), ymin = min(sp->bounds[1], sq->bounds[1]);
  const int xmax = max(sp->bounds[2], sq->bounds[2]), ymax = max(sp->bounds[3], sq->bounds[3]);
  const int k = 3 + lane;
  double cost = 1e300;
  if (!empty && k <= 30) {
    const double ncx = (double)(((xmax - 1) >> k) - (xmin >> k) + 1);
    const double ncy = (double)(((ymax - 1) >> k) - (ymin >> k) + 1);
    const double C = ncx * ncy;
    double bp, ep, bq, eq;
    set_entries(sp, k, bp, ep);
    set_entries(sq, k, bq, eq);
    if (C <= (double)ccap && bq <= (double)ecap) cost = ep + eq + 0.25 * C + ep * eq / C;
  }
  // argmin (ties -> smaller k); k = 30 is always feasible
  int best = k <= 30 ? k : 30;
  double bc = cost;
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const int ok = __shfl_xor_sync(0xffffffffu, best, o);
    if (oc < bc || (oc == bc && ok < best)) {
      bc = oc;
      best = ok;
    }
  }
  if (lane == 0) {
    Grid r{30, 0, 0, 1, 1, 0};
    if (empty) {
      r.empty = 1;
    } else {
      r.k = bc < 1e300 ? best : 30;
      r.cx0 = xmin >> r.k;
      r.cy0 = ymin >> r.k;
      r.ncx = ((xmax - 1) >> r.k) - r.cx0 + 1;
      r.ncy = ((ymax - 1) >> r.k) - r.cy0 + 1;
    }
    *g = r;
  }
}

__global__ void grid_count_kernel(const int4* __restrict__ mq, int64_t nq, const Grid* __restrict__ gp,
                                  int* __restrict__ cell_count) {
  const Grid g = *gp;
  if (g.empty) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x) {
    const int4 m = mq[i];
    if (mbr_empty(m)) continue;
    for (int cy = m.y >> g.k; cy <= (m.w - 1) >> g.k; cy++)
      for (int cx = m.x >> g.k; cx <= (m.z - 1) >> g.k; cx++) atomicAdd(&cell_count[(cy - g.cy0) * g.ncx + cx - g.cx0], 1);
  }
}

// Fill: counts are decremented back to zero as slots are taken, so the count
// array needs no second memset.
__global__ void grid_fill_kernel(const int4* __restrict__ mq, int64_t nq, const Grid* __restrict__ gp,
                                 const int* __restrict__ cell_start, int* __restrict__ cell_count,
                                 int* __restrict__ items) {
  const Grid g = *gp;
  if (g.empty) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x) {
    const int4 m = mq[i];
    if (mbr_empty(m)) continue;
    for (int cy = m.y >> g.k; cy <= (m.w - 1) >> g.k; cy++)
      for (int cx = m.x >> g.k; cx <= (m.z - 1) >> g.k; cx++) {
        const int c = (cy - g.cy0) * g.ncx + cx - g.cx0;
        items[cell_start[c] + atomicSub(&cell_count[c], 1) - 1] = (int)i;
      }
  }
}

// Probe: for each p, visit its cells; a pair is owned by the cell that holds
// its reference point (max xlo, max ylo).  WRITE=false counts, WRITE=true
// writes the segment then insertion-sorts it by q.
template <bool WRITE>
__global__ void probe_kernel(const int4* __restrict__ mp, int64_t np, const int4* __restrict__ mq,
                             const Grid* __restrict__ gp, const int* __restrict__ cell_start,
                             const int* __restrict__ items, long long* __restrict__ count,
                             const long long* __restrict__ start, int2* __restrict__ pairs, long long cap) {
  const Grid g = *gp;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < np; p += int64_t(gridDim.x) * blockDim.x) {
    const int4 a = mp[p];
    long long n = 0;
    if (!g.empty && !mbr_empty(a) && (!WRITE || start[p + 1] <= cap)) {
      const long long base = WRITE ? start[p] : 0;
      for (int cy = a.y >> g.k; cy <= (a.w - 1) >> g.k; cy++)
        for (int cx = a.x >> g.k; cx <= (a.z - 1) >> g.k; cx++) {
          const int c = (cy - g.cy0) * g.ncx + cx - g.cx0;
          for (int it = cell_start[c], e = cell_start[c + 1]; it < e; it++) {
            const int q = items[it];
            const int4 b = mq[q];
            if (a.x < b.z && b.x < a.z && a.y < b.w && b.y < a.w && g.cell(max(a.x, b.x), max(a.y, b.y)) == c) {
              if (WRITE) pairs[base + n] = make_int2((int)p, q);
              n++;
            }
          }
        }
      if (WRITE) {  // insertion sort of the segment by q (segments are short)
        for (long long i = 1; i < n; i++) {
          const int2 v = pairs[base + i];
          long long j = i - 1;
          while (j >= 0 && pairs[base + j].y > v.y) {
            pairs[base + j + 1] = pairs[base + j];
            j--;
          }
          pairs[base + j + 1] = v;
        }
      }
    }
    if (!WRITE) count[p] = n;
  }
}

// --------------------------------------------------------------------- host
static size_t cub_scan_bytes(int64_t n) {
  size_t b32 = 0, b64 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b32, (const int*)nullptr, (int*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b64, (const long long*)nullptr, (long long*)nullptr, (int)n);
  return b32 > b64 ? b32 : b64;
}

struct FilterWs {
  Grid* grid;
  int *cell_count, *cell_start, *items;
  long long *pcount, *pstart;
  void* tmp;
  size_t tmp_bytes;
};

static size_t filter_layout(int64_t np, int64_t nq, Carve& cv, FilterWs& w) {
  const int64_t C = cell_cap(np, nq), E = entry_cap(nq);
  w.grid = cv.take<Grid>(1);
  w.cell_count = cv.take<int>(C + 1);
  w.cell_start = cv.take<int>(C + 1);
  w.items = cv.take<int>(E);
  w.pcount = cv.take<long long>(np + 1);
  w.pstart = cv.take<long long>(np + 1);
  w.tmp_bytes = cub_scan_bytes((C + 1) > (np + 1) ? (C + 1) : (np + 1));
  w.tmp = cv.take<char>(w.tmp_bytes);
  return cv.used;
}

size_t filter_ws_bytes(int64_t np, int64_t nq) {
  Carve cv{nullptr, ~size_t(0)};
  FilterWs w;
  return filter_layout(np, nq, cv, w) + 256;
}

static int blocks_for(int64_t n, int threads) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * (2048 / threads);  // a full SM of threads (these kernels are latency-bound)
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

// Enqueue everything up to the per-P pair offsets (grid, buckets, counts, scan).
static int filter_enqueue(const sccg_polyset* P, const sccg_polyset* Q, FilterWs& w, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  const int4* mp = reinterpret_cast<const int4*>(P->mbr);
  const int4* mq = reinterpret_cast<const int4*>(Q->mbr);
  const int64_t C = cell_cap(np, nq);
  // 1. grid size from the prep statistics (device side), bucket Q
  grid_select_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const SetStats*>(P->stats),
                                           reinterpret_cast<const SetStats*>(Q->stats), C, entry_cap(nq), w.grid);
  cudaMemsetAsync(w.cell_count, 0, sizeof(int) * (C + 1), stream);
  if (nq > 0) grid_count_kernel<<<blocks_for(nq, 256), 256, 0, stream>>>(mq, nq, w.grid, w.cell_count);
  cub::DeviceScan::ExclusiveSum(w.tmp, w.tmp_bytes, w.cell_count, w.cell_start, (int)(C + 1), stream);
  if (nq > 0)
    grid_fill_kernel<<<blocks_for(nq, 256), 256, 0, stream>>>(mq, nq, w.grid, w.cell_start, w.cell_count, w.items);
  // 2. probe: count, scan
  if (np > 0)
    probe_kernel<false><<<blocks_for(np, 128), 128, 0, stream>>>(mp, np, mq, w.grid, w.cell_start, w.items, w.pcount,
                                                                  nullptr, nullptr, 0);
  cudaMemsetAsync(w.pcount + np, 0, sizeof(long long), stream);
  cub::DeviceScan::ExclusiveSum(w.tmp, w.tmp_bytes, w.pcount, w.pstart, (int)(np + 1), stream);
  return check_cuda(cudaGetLastError(), "filter enqueue");
}

static void probe_write(const sccg_polyset* P, const sccg_polyset* Q, FilterWs& w, int32_t* pairs, int64_t cap,
                        cudaStream_t stream) {
  const int64_t np = P->n_polygons;
  if (np > 0 && pairs && cap > 0)
    probe_kernel<true><<<blocks_for(np, 128), 128, 0, stream>>>(
        reinterpret_cast<const int4*>(P->mbr), np, reinterpret_cast<const int4*>(Q->mbr), w.grid, w.cell_start,
        w.items, nullptr, w.pstart, reinterpret_cast<int2*>(pairs), cap);
}

int filter_pairs(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap, int64_t* n_pairs_host,
                 void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  FilterWs w;
  filter_layout(np, nq, cv, w);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "filter workspace too small (see sccg_filter_workspace_bytes)");
  if (int r = filter_enqueue(P, Q, w, stream)) return r;
  // the one host synchronisation: pair count and both sets' prep status
  long long total = 0;
  uint32_t sp[2] = {0, 0}, sq[2] = {0, 0};
  if (int r = check_cuda(cudaMemcpyAsync(&total, w.pstart + np, sizeof(long long), cudaMemcpyDeviceToHost, stream),
                         "count copy"))
    return r;
  if (int r = check_cuda(cudaMemcpyAsync(sp, P->status, 8, cudaMemcpyDeviceToHost, stream), "status copy")) return r;
  if (int r = check_cuda(cudaMemcpyAsync(sq, Q->status, 8, cudaMemcpyDeviceToHost, stream), "status copy")) return r;
  if (int r = check_cuda(cudaStreamSynchronize(stream), "filter sync")) return r;
  for (int s = 0; s < 2; s++) {
    const uint32_t* st = s ? sq : sp;
    if (st[0]) {
      const int code = (st[0] & SCCG_STATUS_ARG) ? SCCG_E_ARG
                       : (st[0] & SCCG_STATUS_NOT_RECTILINEAR) ? SCCG_E_NOT_RECTILINEAR
                                                                : SCCG_E_RANGE;
      return set_error(code, s ? "invalid polygon in set q (sccg_prep status)" : "invalid polygon in set p (sccg_prep status)",
                       (int64_t)st[1]);
    }
  }
  *n_pairs_host = total;
  if (pairs == nullptr || cap < total) return set_error(SCCG_E_CAPACITY, "pair buffer too small", total);
  // write, segment-sorted by q
  if (total > 0) probe_write(P, Q, w, pairs, cap, stream);
  return check_cuda(cudaGetLastError(), "probe write");
}

__global__ void filter_result_kernel(const long long* __restrict__ total, const uint32_t* __restrict__ sp,
                                     const uint32_t* __restrict__ sq, long long* result) {
  if (threadIdx.x == 0) {
    result[0] = *total;
    result[1] = (long long)(sp[0] | sq[0]);
  }
}

int filter_pairs_async(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap,
                       int64_t* result_dev, void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  FilterWs w;
  filter_layout(np, nq, cv, w);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "filter workspace too small (see sccg_filter_workspace_bytes)");
  if (int r = filter_enqueue(P, Q, w, stream)) return r;
  probe_write(P, Q, w, pairs, cap, stream);
  filter_result_kernel<<<1, 32, 0, stream>>>(w.pstart + np, P->status, Q->status,
                                             reinterpret_cast<long long*>(result_dev));
  return check_cuda(cudaGetLastError(), "filter async");
}

}  // namespace sccg
