// join.cu -- MBR-overlap join by a uniform grid hash.
//
// The paper's filter stage searches a Hilbert R-tree on one CPU thread
// (§4.1) to produce "an array of polygon pairs with intersecting
// MBRs"; the predicate is the `&&` MBR test of Fig. 1(b), here
// half-open (reading R4).  On the GPU a uniform grid of 2^k-pixel cells is
// cheaper: Q's MBRs are bucketed into every cell they cover, each P MBR probes
// its cells, and a pair is emitted only from the cell holding its reference
// point (max xlo, max ylo) so it is found exactly once.  Each P's pairs are
// written to its own segment (one-pass probe with a decoupled look-back scan
// of per-P counts) and sorted by q in place, so the output is sorted by (p, q)
// without a global sort.
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
// `grow` = 1: the boxes are grown by one pixel on the high side (closed join).
__device__ __forceinline__ void set_entries(const SetStats* s, int k, int grow, double& bound, double& expect) {
  const double c = 1.0 / (double)(1ll << k), n = (double)s->nonempty;
  const double sw = (double)s->sw + grow * n, sh = (double)s->sh + grow * n;
  const double swh = (double)s->swh + grow * ((double)s->sw + (double)s->sh + n);
  const double cont = swh * c * c + 2.0 * (sw + sh) * c + 4.0 * n;
  const double ext = n * (double)(((s->maxext[0] - 1 + grow) >> k) + 2) * (double)(((s->maxext[1] - 1 + grow) >> k) + 2);
  bound = cont < ext ? cont : ext;
  expect = n + (sw + sh) * c + swh * c * c;
}

// Cell size 2^k minimising the expected work E_p + E_q + C/4 + E_p E_q / C
// (bucket inserts + probes + scan + candidate tests) subject to the workspace
// caps on cells C and (upper-bounded) Q-entries.  Always feasible: once 2^k
// exceeds the largest MBR extent each MBR covers at most 2 x 2 cells.
__global__ void grid_select_kernel(const SetStats* __restrict__ sp, const SetStats* __restrict__ sq, long long ccap,
                                   long long ecap, int grow, Grid* g, int4* __restrict__ zero, long long zero_n4) {
  pdl_trigger();
  // every CTA clears its share of the cell counts (zero_n4 int4s) ...
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < zero_n4; i += (long long)gridDim.x * blockDim.x)
    zero[i] = make_int4(0, 0, 0, 0);
  pdl_wait();  // prep's statistics (and, for what follows, everything before)
  // ... and CTA 0's first warp picks the cell size: lane j evaluates k = 3 + j
  // (k <= 30), then an argmin over lanes
  const int lane = threadIdx.x & 31;
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const bool empty = sp->nonempty == 0 || sq->nonempty == 0;
  const int xmin = min(sp->bounds[0], sq->bounds[0]), ymin = min(sp->bounds[1], sq->bounds[1]);
  const int xmax = max(sp->bounds[2], sq->bounds[2]) + grow, ymax = max(sp->bounds[3], sq->bounds[3]) + grow;
  const int k = 3 + lane;
  double cost = 1e300;
  if (!empty && k <= 30) {
    const double ncx = (double)(((xmax - 1) >> k) - (xmin >> k) + 1);
    const double ncy = (double)(((ymax - 1) >> k) - (ymin >> k) + 1);
    const double C = ncx * ncy;
    double bp, ep, bq, eq;
    set_entries(sp, k, grow, bp, ep);
    set_entries(sq, k, grow, bq, eq);
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

// MBRs covering more than kCoopCells cells (a gland among nuclei, C3) are
// handled by their whole warp, lanes spread over the cells, so one polygon is
// not a serial critical path of hundreds of dependent cell visits.
#ifndef SCCG_COOP_CELLS
#define SCCG_COOP_CELLS 4
#endif
constexpr int kCoopCells = SCCG_COOP_CELLS;

__device__ __forceinline__ int mbr_cells(const int4& m, int k) {
  return (((m.z - 1) >> k) - (m.x >> k) + 1) * (((m.w - 1) >> k) - (m.y >> k) + 1);
}

// Bucket Q: COUNT (FILL = false) adds one per covered cell; FILL takes a slot
// per covered cell (counts are decremented back to zero as slots are taken,
// so the count array needs no second memset) and stores q and its MBR there.
template <bool FILL>
__global__ void grid_bucket_kernel(const int4* __restrict__ mq, int64_t nq, const Grid* __restrict__ gp,
                                   const int* __restrict__ cell_start, int* __restrict__ cell_count,
                                   int* __restrict__ items, int4* __restrict__ item_mbr, int grow) {
  pdl_trigger();
  pdl_wait();
  const Grid g = *gp;
  if (g.empty) return;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  auto insert = [&](int c, int q, const int4& m) {
    if (FILL) {
      const int slot = cell_start[c] + atomicSub(&cell_count[c], 1) - 1;
      items[slot] = q;
      item_mbr[slot] = m;  // the probe tests MBRs straight from the cell's entries
    } else {
      atomicAdd(&cell_count[c], 1);
    }
  };
  for (int64_t base = wid * 32; base < nq; base += nw * 32) {  // warp-uniform trip count
    const int64_t i = base + lane;
    int4 m = make_int4(0, 0, 0, 0);
    bool ok = false;
    if (i < nq) {
      m = mq[i];
      ok = !mbr_empty(m);
      m.z += grow;  // closed join: boxes grown by one pixel on the high side
      m.w += grow;
    }
    const bool coop = ok && mbr_cells(m, g.k) > kCoopCells;
    if (ok && !coop)
      for (int cy = m.y >> g.k; cy <= (m.w - 1) >> g.k; cy++)
        for (int cx = m.x >> g.k; cx <= (m.z - 1) >> g.k; cx++) insert((cy - g.cy0) * g.ncx + cx - g.cx0, (int)i, m);
    for (unsigned bm = __ballot_sync(0xffffffffu, coop); bm; bm &= bm - 1) {
      const int j = __ffs(bm) - 1;
      const int4 mj = make_int4(__shfl_sync(0xffffffffu, m.x, j), __shfl_sync(0xffffffffu, m.y, j),
                                __shfl_sync(0xffffffffu, m.z, j), __shfl_sync(0xffffffffu, m.w, j));
      const int qj = (int)(base + j);
      const int x0 = mj.x >> g.k, y0 = mj.y >> g.k, w = ((mj.z - 1) >> g.k) - x0 + 1;
      const int nc = w * (((mj.w - 1) >> g.k) - y0 + 1);
      for (int t = lane; t < nc; t += 32) insert((y0 + t / w - g.cy0) * g.ncx + x0 + t % w - g.cx0, qj, mj);
    }
  }
}

#ifndef SCCG_PROBE_TILE
#define SCCG_PROBE_TILE 128
#endif
constexpr int kProbeTile = SCCG_PROBE_TILE;  // p per probe CTA

constexpr int kKeep = 4;  // hits kept in registers by the counting pass

// Visit p's cells; count the pairs it owns.  WRITE: store them to out[0..n);
// otherwise keep the first kKeep q indices in keep[].  Entries are tested four
// at a time (independent 16-byte loads in flight).
__device__ __forceinline__ bool owns(const int4& a, const int4& b, int k, int cx0, int cy0, int ncx, int c) {
  return a.x < b.z && b.x < a.z && a.y < b.w && b.y < a.w &&
         ((max(a.y, b.y) >> k) - cy0) * ncx + ((max(a.x, b.x) >> k) - cx0) == c;
}

template <bool WRITE>
__device__ __forceinline__ int probe_cells(const int4& a, long long p, const Grid& gr, const int* __restrict__ cell_start,
                                           const int* __restrict__ items, const int4* __restrict__ item_mbr,
                                           int2* __restrict__ out, int4& keep) {
  const int k = gr.k, cx0 = gr.cx0, cy0 = gr.cy0, ncx = gr.ncx;
  int n = 0;
  int4 kp = keep;
#define SCCG_TAKE(IT)                          \
  {                                            \
    const int q = items[IT];                   \
    if (WRITE) {                               \
      out[n] = make_int2((int)p, q);           \
    } else {                                   \
      kp.x = n == 0 ? q : kp.x;                \
      kp.y = n == 1 ? q : kp.y;                \
      kp.z = n == 2 ? q : kp.z;                \
      kp.w = n == 3 ? q : kp.w;                \
    }                                          \
    n++;                                       \
  }
  for (int cy = a.y >> k; cy <= (a.w - 1) >> k; cy++)
    for (int cx = a.x >> k; cx <= (a.z - 1) >> k; cx++) {
      const int c = (cy - cy0) * ncx + cx - cx0;
      int it = cell_start[c];
      const int e = cell_start[c + 1];
      for (; it + 4 <= e; it += 4) {
        const int4 b0 = item_mbr[it], b1 = item_mbr[it + 1], b2 = item_mbr[it + 2], b3 = item_mbr[it + 3];
        if (owns(a, b0, k, cx0, cy0, ncx, c)) SCCG_TAKE(it)
        if (owns(a, b1, k, cx0, cy0, ncx, c)) SCCG_TAKE(it + 1)
        if (owns(a, b2, k, cx0, cy0, ncx, c)) SCCG_TAKE(it + 2)
        if (owns(a, b3, k, cx0, cy0, ncx, c)) SCCG_TAKE(it + 3)
      }
      for (; it < e; it++)
        if (owns(a, item_mbr[it], k, cx0, cy0, ncx, c)) SCCG_TAKE(it)
    }
#undef SCCG_TAKE
  keep = kp;
  return n;
}

__device__ __forceinline__ int4 shfl4(const int4& v, int j) {
  return make_int4(__shfl_sync(0xffffffffu, v.x, j), __shfl_sync(0xffffffffu, v.y, j), __shfl_sync(0xffffffffu, v.z, j),
                   __shfl_sync(0xffffffffu, v.w, j));
}

// A big MBR probed by its whole warp.  Its cell rectangle is taken 32 cells
// at a time (lane l reads cell l's entry range); the entries of those cells
// are then flattened over the lanes (a warp scan of the range lengths, and a
// 5-step shuffle search for each entry's cell), so a lane tests entry after
// entry of ALL the cells with independent loads -- a gland whose cells hold
// dozens of nuclei each (C3) is not a serial walk per cell.  COUNT returns the
// pairs it owns (every lane gets the total); WRITE appends them to seg[] in
// arbitrary order (slots from *fill, reset here) -- the q order is restored
// by the segment sort.
template <bool WRITE>
__device__ int coop_cells(const int4 a, long long p, const Grid& g, const int* __restrict__ cell_start,
                          const int* __restrict__ items, const int4* __restrict__ item_mbr, int2* __restrict__ seg,
                          int* fill) {
  const int lane = threadIdx.x & 31;
  const int k = g.k, cx0 = g.cx0, cy0 = g.cy0, ncx = g.ncx;
  const int x0 = a.x >> k, y0 = a.y >> k, w = ((a.z - 1) >> k) - x0 + 1;
  const int nc = w * (((a.w - 1) >> k) - y0 + 1);
  if (WRITE) {
    if (lane == 0) *fill = 0;
    __syncwarp();
  }
  int cnt = 0;
  for (int base = 0; base < nc; base += 32) {  // warp-uniform
    const int t = base + lane;
    int c = 0, s = 0, len = 0;
    if (t < nc) {
      c = (y0 + t / w - cy0) * ncx + (x0 + t % w - cx0);
      s = cell_start[c];
      len = cell_start[c + 1] - s;
    }
    int incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - len;
    for (int f0 = 0; f0 < total; f0 += 32) {  // warp-uniform
      const int f = f0 + lane;
      int j = 0;  // the lane whose cell holds flattened entry f: #lanes with incl <= f
      for (int b = 16; b; b >>= 1)
        if (__shfl_sync(0xffffffffu, incl, j + b - 1) <= f) j += b;
      const int cj = __shfl_sync(0xffffffffu, c, j), sj = __shfl_sync(0xffffffffu, s, j);
      const int ej = __shfl_sync(0xffffffffu, excl, j);
      if (f < total) {
        const int it = sj + (f - ej);
        if (owns(a, item_mbr[it], k, cx0, cy0, ncx, cj)) {
          if (WRITE) seg[atomicAdd(fill, 1)] = make_int2((int)p, items[it]);
          cnt++;
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  return cnt;
}

// Sort seg[0..n) by q (distinct within a segment) with the warp: a bitonic
// network in its ascending-only form (each merge starts by comparing i with
// its mirror i ^ (k - 1)), so positions >= n behave as +inf and are never
// touched -- no padding needed.  Up to kSortBuf keys are sorted in a shared
// buffer (one per CTA, under a lock -- long segments are rare; kept small so
// the L1 the probe lives on stays large); longer segments in place in global
// memory (L1/L2-resident).
constexpr int kSortBuf = 1024;
constexpr int kThreadSortMax = 32;  // segments up to this length: the owning thread sorts

template <typename Key, typename Get, typename Put>
__device__ __forceinline__ void warp_bitonic(int n, Get get, Put put) {
  const int lane = threadIdx.x & 31;
  int m = 1;
  while (m < n) m <<= 1;
  for (int k = 2; k <= m; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < m; i += 32) {
        const int l = j == (k >> 1) ? (i ^ (k - 1)) : (i ^ j);  // mirror first, then halves
        if (l > i && l < n) {
          const Key u = get(i), v = get(l);
          if (v < u) {
            put(i, v);
            put(l, u);
          }
        }
      }
      __syncwarp();
    }
}

__device__ void warp_sort_segment(int2* seg, int n, int* buf, int* lock) {
  const int lane = threadIdx.x & 31;
  if (n <= 1) return;
  if (n <= kSortBuf) {
    if (lane == 0)
      while (atomicCAS(lock, 0, 1) != 0) {
      }
    __syncwarp();
    const int p = seg[0].x;
    for (int i = lane; i < n; i += 32) buf[i] = seg[i].y;
    __syncwarp();
    warp_bitonic<int>(n, [&](int i) { return buf[i]; }, [&](int i, int v) { buf[i] = v; });
    for (int i = lane; i < n; i += 32) seg[i] = make_int2(p, buf[i]);
    __threadfence_block();
    __syncwarp();
    if (lane == 0) atomicExch(lock, 0);
  } else {
    const int p = seg[0].x;
    __syncwarp();
    warp_bitonic<int>(n, [&](int i) { return seg[i].y; }, [&](int i, int v) { seg[i] = make_int2(p, v); });
  }
  __syncwarp();
}

// Probe, per CTA tile of kProbeTile consecutive p (thread per p).  A pair is
// owned by the cell that holds its reference point (max xlo, max ylo).  Each
// thread counts its pairs (keeping up to kKeep hits in registers; MBRs over
// many cells are counted by their whole warp) and the CTA scans the counts.
// BUCKET pass: the tile writes its (p, q)-sorted pairs into its own bucket of
// kBucket slots (no cross-CTA dependency) and records its count.  COMPACT pass:
// each tile sums the preceding tiles' counts (all known by then; a few
// vectorized L2 loads per thread) for its offset, copies its bucket there, or
// -- when the tile overflowed its bucket -- probes again and writes there
// directly; the last tile writes the total (and the async result word).  Pairs
// past `cap` are not written; the total is exact.
constexpr int kBucket = 1024;
#ifndef SCCG_PROBE_MINB
#define SCCG_PROBE_MINB 12
#endif

template <bool COMPACT>
__global__ void __launch_bounds__(kProbeTile, SCCG_PROBE_MINB) probe_kernel(const int4* __restrict__ mp, int64_t np,
                                                           const Grid* __restrict__ gp,
                                                           const int* __restrict__ cell_start,
                                                           const int* __restrict__ items,
                                                           const int4* __restrict__ item_mbr,
                                                           int* __restrict__ tile_cnt,
                                                           unsigned char* __restrict__ tile_long,
                                                           int2* __restrict__ bucket, int2* __restrict__ pairs,
                                                           long long cap, long long* __restrict__ total,
                                                           long long* __restrict__ result,
                                                           const uint32_t* __restrict__ status_p,
                                                           const uint32_t* __restrict__ status_q, int grow) {
  __shared__ int s_warp[kProbeTile / 32];
  __shared__ long long s_sum[kProbeTile / 32];
  __shared__ int s_fill[kProbeTile / 32];
  __shared__ int s_coop[kProbeTile];     // threads of this tile whose MBR the warps probe together
  __shared__ int s_coopval[kProbeTile];  // ... their pair count, then their output offset
  __shared__ int s_cw[kProbeTile / 32];
  __shared__ int s_sort[kSortBuf];
  __shared__ int s_lock;
  __shared__ int2 s_pairs[COMPACT ? kBucket : 1];      // compaction: the tile's bucket
  __shared__ unsigned s_head[COMPACT ? kBucket / 32 : 1];  // ... first pair of each p
  __shared__ int s_runs[COMPACT ? 2 * kProbeTile + 1 : 1];  // ... long runs (start, length), count
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  int2* dst;  // this tile's output: its bucket, or its final place
  if (COMPACT) {
    long long sum = 0;  // this tile's offset: the preceding tiles' counts
    const int4* c4 = reinterpret_cast<const int4*>(tile_cnt);
    for (int i = threadIdx.x; i < (tile >> 2); i += kProbeTile) {
      const int4 v = c4[i];
      sum += (long long)v.x + v.y + v.z + v.w;
    }
    for (int i = (tile & ~3) + threadIdx.x; i < tile; i += kProbeTile) sum += tile_cnt[i];
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_sum[warp] = sum;
    __syncthreads();
    long long off = 0;
    for (int w = 0; w < kProbeTile / 32; w++) off += s_sum[w];
    const int cnt = tile_cnt[tile];
    if (tile == (int)gridDim.x - 1 && threadIdx.x == 0) {
      *total = off + cnt;
      if (result) {
        result[0] = off + cnt;
        result[1] = (long long)(status_p[0] | status_q[0]);
      }
    }
    if (cnt == 0 || pairs == nullptr || off + cnt > cap) return;
    if (cnt <= kBucket && !tile_long[tile]) {  // copy the bucket
      const int2* src = bucket + (size_t)tile * kBucket;
      for (int i = threadIdx.x; i < cnt; i += kProbeTile) pairs[off + i] = src[i];
      return;
    }
    if (cnt <= kBucket) {
      // stage the bucket; runs of one p longer than kThreadSortMax were left
      // unsorted by the bucket pass -- the whole CTA sorts each by q here
      const int2* src = bucket + (size_t)tile * kBucket;
      for (int i = threadIdx.x; i < kBucket / 32; i += kProbeTile) s_head[i] = 0u;
      if (threadIdx.x == 0) s_runs[2 * kProbeTile] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += kProbeTile) {
        const int2 v = src[i];
        s_pairs[i] = v;
        if (i == 0 || src[i - 1].x != v.x) atomicOr(&s_head[i >> 5], 1u << (i & 31));
      }
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += kProbeTile) {
        if (!((s_head[i >> 5] >> (i & 31)) & 1u)) continue;
        int e = i + 1;  // next head (or the end)
        while (e < cnt) {
          const unsigned w = s_head[e >> 5] >> (e & 31);
          if (w) {
            e += __ffs(w) - 1;
            break;
          }
          e = (e | 31) + 1;
        }
        if (e > cnt) e = cnt;
        if (e - i > kThreadSortMax) {
          const int r = atomicAdd(&s_runs[2 * kProbeTile], 1);
          s_runs[2 * r] = i;
          s_runs[2 * r + 1] = e - i;
        }
      }
      __syncthreads();
      const int nruns = s_runs[2 * kProbeTile];
      for (int i = threadIdx.x; i < cnt; i += kProbeTile) pairs[off + i] = s_pairs[i];
      if (nruns == 0) return;
      __syncthreads();  // the long runs' unsorted copies are overwritten below
      // long runs: rank sort -- an entry's place in its run is the number of
      // the run's q below its own (q are distinct within a run); every thread
      // moves on to the next run without a barrier, so a tile with many glands
      // costs its total run work, not a barrier-bound network per run
      for (int r = 0; r < nruns; r++) {
        const int s0 = s_runs[2 * r], n = s_runs[2 * r + 1];
        const int2* run = s_pairs + s0;
        for (int i = threadIdx.x; i < n; i += kProbeTile) {
          const int2 v = run[i];
          int rank = 0;
#pragma unroll 4
          for (int j = 0; j < n; j++) rank += run[j].y < v.y ? 1 : 0;
          pairs[off + s0 + rank] = v;
        }
      }
      return;
    }
    dst = pairs + off;  // overflowed tile: probe again, write in place
  } else {
    dst = bucket + (size_t)tile * kBucket;
  }
  if (threadIdx.x == 0) s_lock = 0;
  const int64_t p = (int64_t)tile * kProbeTile + threadIdx.x;
  const Grid g = *gp;
  int4 a = make_int4(0, 0, 0, 0);
  const bool live = p < np && !g.empty;
  if (live) a = mp[p];
  const bool act = live && !mbr_empty(a);
  a.z += grow;  // closed join: boxes grown by one pixel on the high side
  a.w += grow;
  int4 keep = make_int4(0, 0, 0, 0);
  const bool coop = act && mbr_cells(a, g.k) > kCoopCells;  // big MBR: its warp probes it together
  int n = act && !coop ? probe_cells<false>(a, p, g, cell_start, items, item_mbr, nullptr, keep) : 0;
  // big MBRs of the whole tile (glands among nuclei, C3: often consecutive in
  // p) are dealt round-robin to the tile's warps, so their serial cell walks
  // run side by side instead of queueing on the one warp that holds them
  int ncoop = 0;
  if (__syncthreads_or(coop)) {
    const unsigned cm = __ballot_sync(0xffffffffu, coop);
    if (lane == 0) s_cw[warp] = __popc(cm);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < kProbeTile / 32; w++) {
      off += w < warp ? s_cw[w] : 0;
      ncoop += s_cw[w];
    }
    if (coop) s_coop[off + __popc(cm & lanemask_lt())] = threadIdx.x;
    __syncthreads();
    for (int t = warp; t < ncoop; t += kProbeTile / 32) {
      const int j = s_coop[t];
      int4 aj = mp[(int64_t)tile * kProbeTile + j];
      aj.z += grow;
      aj.w += grow;
      const int cnt = coop_cells<false>(aj, (int64_t)tile * kProbeTile + j, g, cell_start, items, item_mbr, nullptr,
                                        nullptr);
      if (lane == 0) s_coopval[j] = cnt;
    }
    __syncthreads();
    if (coop) n = s_coopval[threadIdx.x];
  }
  // CTA exclusive scan of the counts
  int x = n;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  int wbase = 0, agg = 0;
  for (int w = 0; w < kProbeTile / 32; w++) {
    const int v = s_warp[w];
    wbase += w < warp ? v : 0;
    agg += v;
  }
  const int base = wbase + x - n;
  if (!COMPACT) {
    if (threadIdx.x == 0) tile_cnt[tile] = agg;
    if (agg > kBucket) return;  // rare: the compact pass probes this tile again
  }
  const bool fits = n > 0;
  // big MBRs: gathered by the warps (round-robin as above), unsorted
  if (ncoop > 0) {
    if (coop) s_coopval[threadIdx.x] = fits ? base : -1;
    __syncthreads();
    for (int t = warp; t < ncoop; t += kProbeTile / 32) {
      const int j = s_coop[t];
      if (s_coopval[j] < 0) continue;  // warp-uniform
      int4 aj = mp[(int64_t)tile * kProbeTile + j];
      aj.z += grow;
      aj.w += grow;
      coop_cells<true>(aj, (int64_t)tile * kProbeTile + j, g, cell_start, items, item_mbr, dst + s_coopval[j],
                       &s_fill[warp]);
    }
    __syncthreads();  // the warps' writes are visible to the segment's own thread
    if (coop && fits && n <= kThreadSortMax) {  // short segment: its thread sorts it by q (longer: see below)
      int2* seg = dst + base;
      for (int i = 1; i < n; i++) {
        const int2 v = seg[i];
        int j = i - 1;
        while (j >= 0 && seg[j].y > v.y) {
          seg[j + 1] = seg[j];
          j--;
        }
        seg[j + 1] = v;
      }
    }
  }
  if (fits && !coop) {
    int2* seg = dst + base;
    if (n <= kKeep) {  // the counting pass kept them: sort in registers, write
      const int big = 0x7fffffff;  // pad the unused slots so a 4-sorting network applies
      int k0 = keep.x, k1 = n > 1 ? keep.y : big, k2 = n > 2 ? keep.z : big, k3 = n > 3 ? keep.w : big;
#define SCCG_CSWAP(U, V)        \
  {                             \
    const int lo = min(U, V);   \
    V = max(U, V);              \
    U = lo;                     \
  }
      SCCG_CSWAP(k0, k1)
      SCCG_CSWAP(k2, k3)
      SCCG_CSWAP(k0, k2)
      SCCG_CSWAP(k1, k3)
      SCCG_CSWAP(k1, k2)
#undef SCCG_CSWAP
      seg[0] = make_int2((int)p, k0);
      if (n > 1) seg[1] = make_int2((int)p, k1);
      if (n > 2) seg[2] = make_int2((int)p, k2);
      if (n > 3) seg[3] = make_int2((int)p, k3);
    } else {
      probe_cells<true>(a, p, g, cell_start, items, item_mbr, seg, keep);
      if (n <= kThreadSortMax)
        for (int i = 1; i < n; i++) {  // insertion sort of a short segment by q
          const int2 v = seg[i];
          int j = i - 1;
          while (j >= 0 && seg[j].y > v.y) {
            seg[j + 1] = seg[j];
            j--;
          }
          seg[j + 1] = v;
        }
    }
  }
  // long segments (big MBRs, or many hits): sorted by the compaction pass for
  // a bucket, here by the warp when writing in place (an overflowed tile)
  if (!COMPACT) {
    const int any_long = __syncthreads_or(fits && n > kThreadSortMax);
    if (threadIdx.x == 0) tile_long[tile] = any_long ? 1 : 0;
    return;
  }
  __syncthreads();  // s_lock initialised; every segment written
  for (unsigned bm = __ballot_sync(0xffffffffu, fits && n > kThreadSortMax); bm; bm &= bm - 1) {
    const int j = __ffs(bm) - 1;
    warp_sort_segment(dst + __shfl_sync(0xffffffffu, base, j), __shfl_sync(0xffffffffu, n, j), s_sort, &s_lock);
  }
}

// --------------------------------------------------------------------- host
static size_t cub_scan_bytes(int64_t n) {
  size_t b32 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b32, (const int*)nullptr, (int*)nullptr, (int)n);
  return b32;
}

static int64_t probe_tiles(int64_t np) { return (np + kProbeTile - 1) / kProbeTile; }

struct FilterWs {
  Grid* grid;
  int *cell_count, *cell_start, *items;
  int4* item_mbr;
  int* tile_cnt;   // [T] pairs per probe tile
  unsigned char* tile_long;  // [T] the tile's bucket holds a segment the compaction sorts
  int2* bucket;    // [T][kBucket] per-tile pair buckets
  long long* total;
  void* tmp;
  size_t tmp_bytes;
};

static size_t filter_layout(int64_t np, int64_t nq, Carve& cv, FilterWs& w) {
  const int64_t C = cell_cap(np, nq), E = entry_cap(nq);
  w.grid = cv.take<Grid>(1);
  w.cell_count = cv.take<int>(C + 1);
  w.cell_start = cv.take<int>(C + 1);
  w.items = cv.take<int>(E);
  w.item_mbr = cv.take<int4>(E);
  const int64_t T = probe_tiles(np);
  w.tile_cnt = cv.take<int>(T + 4);
  w.tile_long = cv.take<unsigned char>(T + 1);
  w.total = cv.take<long long>(1);
  w.bucket = cv.take<int2>(T * kBucket);
  w.tmp_bytes = cub_scan_bytes(C + 1);
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

__global__ void filter_result_kernel(const long long* __restrict__ total, const uint32_t* __restrict__ sp,
                                     const uint32_t* __restrict__ sq, long long* result) {
  if (threadIdx.x == 0) {
    result[0] = *total;
    result[1] = (long long)(sp[0] | sq[0]);
  }
}

// Enqueue the whole join: grid, Q buckets, probe into per-tile buckets, scan
// of the tile counts, compaction (pairs written when they fit in `cap`; the
// exact total always lands in w.total).
static int filter_enqueue(const sccg_polyset* P, const sccg_polyset* Q, FilterWs& w, int32_t* pairs, int64_t cap,
                          long long* result, int grow, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  const int4* mp = reinterpret_cast<const int4*>(P->mbr);
  const int4* mq = reinterpret_cast<const int4*>(Q->mbr);
  const int64_t C = cell_cap(np, nq), T = probe_tiles(np);
  // 1. grid size from the prep statistics (device side) and the count array
  // cleared in the same launch; bucket Q (chained onto it by PDL)
  const long long zero_n4 = (long long)((sizeof(int) * (C + 1) + 15) / 16);  // cell_count's slice is 256-B aligned
  launch_pdl(grid_select_kernel, dim3((unsigned)blocks_for(zero_n4, 256)), dim3(256), 0, stream,
             reinterpret_cast<const SetStats*>(P->stats), reinterpret_cast<const SetStats*>(Q->stats), (long long)C,
             (long long)entry_cap(nq), grow, w.grid, reinterpret_cast<int4*>(w.cell_count), zero_n4);
  if (nq > 0)
    launch_pdl(grid_bucket_kernel<false>, dim3(blocks_for(nq, 256)), dim3(256), 0, stream, mq, nq, w.grid,
               (const int*)nullptr, w.cell_count, (int*)nullptr, (int4*)nullptr, grow);
  cub::DeviceScan::ExclusiveSum(w.tmp, w.tmp_bytes, w.cell_count, w.cell_start, (int)(C + 1), stream);
  if (nq > 0)
    launch_pdl(grid_bucket_kernel<true>, dim3(blocks_for(nq, 256)), dim3(256), 0, stream, mq, nq, w.grid,
               w.cell_start, w.cell_count, w.items, w.item_mbr, grow);
  // 2. probe into tile buckets; compaction (offsets, copies, total)
  if (np > 0) {
    launch_pdl(probe_kernel<false>, dim3((unsigned)T), dim3(kProbeTile), 0, stream, mp, np, w.grid, w.cell_start,
               w.items, w.item_mbr, w.tile_cnt, w.tile_long, w.bucket, (int2*)nullptr, (long long)0,
               (long long*)nullptr, (long long*)nullptr, (const uint32_t*)nullptr, (const uint32_t*)nullptr, grow);
    launch_pdl(probe_kernel<true>, dim3((unsigned)T), dim3(kProbeTile), 0, stream, mp, np, w.grid, w.cell_start,
               w.items, w.item_mbr, w.tile_cnt, w.tile_long, w.bucket, reinterpret_cast<int2*>(pairs),
               (long long)(pairs ? cap : 0), w.total, result, P->status, Q->status, grow);
  } else {
    cudaMemsetAsync(w.total, 0, sizeof(long long), stream);
    if (result) filter_result_kernel<<<1, 32, 0, stream>>>(w.total, P->status, Q->status, result);
  }
  return check_cuda(cudaGetLastError(), "filter enqueue");
}

int filter_pairs(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap, int64_t* n_pairs_host,
                 void* ws, size_t ws_bytes, int closed, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  FilterWs w;
  filter_layout(np, nq, cv, w);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "filter workspace too small (see sccg_filter_workspace_bytes)");
  if (int r = filter_enqueue(P, Q, w, pairs, cap, nullptr, closed ? 1 : 0, stream)) return r;
  // the one host synchronisation: pair count and both sets' prep status
  long long total = 0;
  uint32_t sp[2] = {0, 0}, sq[2] = {0, 0};
  if (int r = check_cuda(cudaMemcpyAsync(&total, w.total, sizeof(long long), cudaMemcpyDeviceToHost, stream),
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
  return SCCG_OK;
}

int filter_pairs_async(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap,
                       int64_t* result_dev, void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  FilterWs w;
  filter_layout(np, nq, cv, w);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "filter workspace too small (see sccg_filter_workspace_bytes)");
  if (int r = filter_enqueue(P, Q, w, pairs, cap, reinterpret_cast<long long*>(result_dev), 0, stream)) return r;
  return check_cuda(cudaGetLastError(), "filter async");
}

}  // namespace sccg
