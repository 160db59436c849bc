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
#include <cub/device/device_scan.cuh>

#include "internal.cuh"

namespace sccg {

constexpr int kKMin = 3, kKMax = 30, kNK = kKMax - kKMin + 1;

struct JoinStats {
  int32_t bounds[4];              // xmin, ymin (atomicMin), xmax, ymax (atomicMax) over non-empty MBRs
  unsigned long long entries[2][32];  // per set, per k: sum of cells covered
};

__device__ __forceinline__ bool mbr_empty(const int4& m) { return m.x >= m.z || m.y >= m.w; }

__global__ void join_stats_kernel(const int4* __restrict__ mp, int64_t np, const int4* __restrict__ mq, int64_t nq,
                                  JoinStats* st) {
  __shared__ unsigned long long s_ent[2][kNK];
  __shared__ int s_b[4];
  for (int i = threadIdx.x; i < 2 * kNK; i += blockDim.x) (&s_ent[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    s_b[0] = s_b[1] = INT_MAX;
    s_b[2] = s_b[3] = INT_MIN;
  }
  __syncthreads();
  int bx0 = INT_MAX, by0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN;
  for (int s = 0; s < 2; s++) {
    const int4* m_ = s == 0 ? mp : mq;
    const int64_t n_ = s == 0 ? np : nq;
    unsigned long long ent[kNK];
#pragma unroll
    for (int k = 0; k < kNK; k++) ent[k] = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_; i += int64_t(gridDim.x) * blockDim.x) {
      const int4 m = m_[i];
      if (mbr_empty(m)) continue;
      bx0 = min(bx0, m.x);
      by0 = min(by0, m.y);
      bx1 = max(bx1, m.z);
      by1 = max(by1, m.w);
#pragma unroll
      for (int k = 0; k < kNK; k++) {
        const int kk = k + kKMin;
        unsigned long long cx = (unsigned)(((m.z - 1) >> kk) - (m.x >> kk) + 1);
        unsigned long long cy = (unsigned)(((m.w - 1) >> kk) - (m.y >> kk) + 1);
        ent[k] += cx * cy;
      }
    }
#pragma unroll
    for (int k = 0; k < kNK; k++) {
      unsigned long long v = ent[k];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_ent[s][k], v);
    }
  }
  bx0 = __reduce_min_sync(0xffffffffu, bx0);
  by0 = __reduce_min_sync(0xffffffffu, by0);
  bx1 = __reduce_max_sync(0xffffffffu, bx1);
  by1 = __reduce_max_sync(0xffffffffu, by1);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_b[0], bx0);
    atomicMin(&s_b[1], by0);
    atomicMax(&s_b[2], bx1);
    atomicMax(&s_b[3], by1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * kNK; i += blockDim.x) {
    unsigned long long v = (&s_ent[0][0])[i];
    if (v) atomicAdd(&st->entries[i / kNK][i % kNK], v);
  }
  if (threadIdx.x == 0) {
    atomicMin(&st->bounds[0], s_b[0]);
    atomicMin(&st->bounds[1], s_b[1]);
    atomicMax(&st->bounds[2], s_b[2]);
    atomicMax(&st->bounds[3], s_b[3]);
  }
}

__global__ void join_stats_init(JoinStats* st) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) (&st->entries[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    st->bounds[0] = st->bounds[1] = INT_MAX;
    st->bounds[2] = st->bounds[3] = INT_MIN;
  }
}

struct Grid {
  int k, cx0, cy0, ncx, ncy;
  __device__ __forceinline__ int cell(int x, int y) const { return ((y >> k) - cy0) * ncx + ((x >> k) - cx0); }
};

__global__ void grid_count_kernel(const int4* __restrict__ mq, int64_t nq, Grid g, int* __restrict__ cell_count) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x) {
    const int4 m = mq[i];
    if (mbr_empty(m)) continue;
    for (int cy = m.y >> g.k; cy <= (m.w - 1) >> g.k; cy++)
      for (int cx = m.x >> g.k; cx <= (m.z - 1) >> g.k; cx++) atomicAdd(&cell_count[(cy - g.cy0) * g.ncx + cx - g.cx0], 1);
  }
}

__global__ void grid_fill_kernel(const int4* __restrict__ mq, int64_t nq, Grid g, const int* __restrict__ cell_start,
                                 int* __restrict__ cell_fill, int* __restrict__ items) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x) {
    const int4 m = mq[i];
    if (mbr_empty(m)) continue;
    for (int cy = m.y >> g.k; cy <= (m.w - 1) >> g.k; cy++)
      for (int cx = m.x >> g.k; cx <= (m.z - 1) >> g.k; cx++) {
        const int c = (cy - g.cy0) * g.ncx + cx - g.cx0;
        items[cell_start[c] + atomicAdd(&cell_fill[c], 1)] = (int)i;
      }
  }
}

// Probe: for each p, visit its cells; a pair is owned by the cell that holds
// its reference point (max xlo, max ylo).  WRITE=false counts, WRITE=true
// writes the segment then insertion-sorts it by q.
template <bool WRITE>
__global__ void probe_kernel(const int4* __restrict__ mp, int64_t np, const int4* __restrict__ mq, Grid g,
                             const int* __restrict__ cell_start, const int* __restrict__ items,
                             long long* __restrict__ count, const long long* __restrict__ start,
                             int2* __restrict__ pairs) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < np; p += int64_t(gridDim.x) * blockDim.x) {
    const int4 a = mp[p];
    long long n = 0;
    if (!mbr_empty(a)) {
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
          int2 v = pairs[base + i];
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
static int64_t cell_cap(int64_t np, int64_t nq) { return 2 * (np + nq) + 1024; }
static int64_t entry_cap(int64_t nq) { return 4 * nq + 1024; }

static size_t cub_scan_bytes(int64_t n) {
  size_t b32 = 0, b64 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b32, (const int*)nullptr, (int*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b64, (const long long*)nullptr, (long long*)nullptr, (int)n);
  return b32 > b64 ? b32 : b64;
}

static size_t filter_layout(int64_t np, int64_t nq, Carve& cv, JoinStats** st, int** cell_count, int** cell_start,
                            int** cell_fill, int** items, long long** pcount, long long** pstart, void** tmp,
                            size_t* tmp_bytes) {
  const int64_t C = cell_cap(np, nq), E = entry_cap(nq);
  *st = cv.take<JoinStats>(1);
  *cell_count = cv.take<int>(C + 1);
  *cell_start = cv.take<int>(C + 1);
  *cell_fill = cv.take<int>(C + 1);
  *items = cv.take<int>(E);
  *pcount = cv.take<long long>(np + 1);
  *pstart = cv.take<long long>(np + 1);
  *tmp_bytes = cub_scan_bytes((C + 1) > (np + 1) ? (C + 1) : (np + 1));
  *tmp = cv.take<char>(*tmp_bytes);
  return cv.used;
}

size_t filter_ws_bytes(int64_t np, int64_t nq) {
  Carve cv{nullptr, ~size_t(0)};
  JoinStats* st;
  int *a, *b, *c, *d;
  long long *e, *f;
  void* t;
  size_t tb;
  return filter_layout(np, nq, cv, &st, &a, &b, &c, &d, &e, &f, &t, &tb) + 256;
}

static int blocks_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sms * 8;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int filter_pairs(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap, int64_t* n_pairs_host,
                 void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  JoinStats* st;
  int *cell_count, *cell_start, *cell_fill, *items;
  long long *pcount, *pstart;
  void* tmp;
  size_t tmp_bytes;
  filter_layout(np, nq, cv, &st, &cell_count, &cell_start, &cell_fill, &items, &pcount, &pstart, &tmp, &tmp_bytes);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "filter workspace too small (see sccg_filter_workspace_bytes)");
  const int4* mp = reinterpret_cast<const int4*>(P->mbr);
  const int4* mq = reinterpret_cast<const int4*>(Q->mbr);

  // 1. bounds + per-k cell-entry counts, then pick the cell size on the host
  join_stats_init<<<1, 64, 0, stream>>>(st);
  if (np + nq > 0) join_stats_kernel<<<blocks_for(np + nq, 256), 256, 0, stream>>>(mp, np, mq, nq, st);
  JoinStats hs;
  uint32_t stat_p[2], stat_q[2];
  if (int r = check_cuda(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, stream), "stats copy")) return r;
  if (int r = check_cuda(cudaMemcpyAsync(stat_p, P->status, 8, cudaMemcpyDeviceToHost, stream), "status copy")) return r;
  if (int r = check_cuda(cudaMemcpyAsync(stat_q, Q->status, 8, cudaMemcpyDeviceToHost, stream), "status copy")) return r;
  if (int r = check_cuda(cudaStreamSynchronize(stream), "filter sync 1")) return r;
  for (int s = 0; s < 2; s++) {
    uint32_t* sp = s ? stat_q : stat_p;
    if (sp[0]) {
      int code = (sp[0] & SCCG_STATUS_ARG) ? SCCG_E_ARG
                 : (sp[0] & SCCG_STATUS_NOT_RECTILINEAR) ? SCCG_E_NOT_RECTILINEAR
                                                          : SCCG_E_RANGE;
      return set_error(code, s ? "invalid polygon in set q (sccg_prep status)" : "invalid polygon in set p (sccg_prep status)",
                       (int64_t)sp[1]);
    }
  }
  const bool empty = hs.bounds[0] > hs.bounds[2] || hs.bounds[1] > hs.bounds[3] || np == 0 || nq == 0 ||
                     hs.entries[0][kNK - 1] == 0 || hs.entries[1][kNK - 1] == 0;
  if (empty) {
    *n_pairs_host = 0;
    return SCCG_OK;
  }
  const int64_t Ccap = cell_cap(np, nq), Ecap = entry_cap(nq);
  int best_k = kKMax;
  double best_cost = 1e300;
  for (int k = kKMin; k <= kKMax; k++) {
    const int64_t ncx = (int64_t)((hs.bounds[2] - 1) >> k) - (hs.bounds[0] >> k) + 1;
    const int64_t ncy = (int64_t)((hs.bounds[3] - 1) >> k) - (hs.bounds[1] >> k) + 1;
    const double C = (double)ncx * (double)ncy;
    const double Ep = (double)hs.entries[0][k - kKMin], Eq = (double)hs.entries[1][k - kKMin];
    if (C > (double)Ccap || Eq > (double)Ecap) continue;
    const double cost = Ep + Eq + 0.25 * C + Ep * Eq / C;
    if (cost < best_cost) {
      best_cost = cost;
      best_k = k;
    }
  }
  Grid g;
  g.k = best_k;
  g.cx0 = hs.bounds[0] >> best_k;
  g.cy0 = hs.bounds[1] >> best_k;
  g.ncx = ((hs.bounds[2] - 1) >> best_k) - g.cx0 + 1;
  g.ncy = ((hs.bounds[3] - 1) >> best_k) - g.cy0 + 1;
  const int C = g.ncx * g.ncy;

  // 2. bucket Q
  cudaMemsetAsync(cell_count, 0, sizeof(int) * (C + 1), stream);
  cudaMemsetAsync(cell_fill, 0, sizeof(int) * (C + 1), stream);
  grid_count_kernel<<<blocks_for(nq, 256), 256, 0, stream>>>(mq, nq, g, cell_count);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cell_count, cell_start, C + 1, stream);
  grid_fill_kernel<<<blocks_for(nq, 256), 256, 0, stream>>>(mq, nq, g, cell_start, cell_fill, items);
  // 3. probe: count, scan, total
  probe_kernel<false><<<blocks_for(np, 128), 128, 0, stream>>>(mp, np, mq, g, cell_start, items, pcount, nullptr,
                                                                nullptr);
  cudaMemsetAsync(pcount + np, 0, sizeof(long long), stream);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, pcount, pstart, (int)(np + 1), stream);
  long long total = 0;
  if (int r = check_cuda(cudaMemcpyAsync(&total, pstart + np, sizeof(total), cudaMemcpyDeviceToHost, stream),
                         "count copy"))
    return r;
  if (int r = check_cuda(cudaStreamSynchronize(stream), "filter sync 2")) return r;
  *n_pairs_host = total;
  if (pairs == nullptr || cap < total) return set_error(SCCG_E_CAPACITY, "pair buffer too small", total);
  // 4. write, segment-sorted by q
  if (total > 0)
    probe_kernel<true><<<blocks_for(np, 128), 128, 0, stream>>>(mp, np, mq, g, cell_start, items, nullptr, pstart,
                                                                 reinterpret_cast<int2*>(pairs));
  return check_cuda(cudaGetLastError(), "probe write");
}

}  // namespace sccg
