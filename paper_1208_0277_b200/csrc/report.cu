// report.cu -- what follows the per-pair areas:
//  * sccg_contains: ST_Contains from the areas (§3.4);
//  * sccg_report: the per-tile SimilarityReport -- pair
//    totals, exact ratio limbs, polygon and missing-polygon counts per
//    tile of the image grid;
//  * sccg_sums_pack / sccg_sums_unpack: the cross-GPU reduction vector of the
//    sums (additive fields + status bits expanded to 0/1 counts).
#include "pixelbox_common.cuh"

namespace sccg {

// ----------------------------------------------------------- ST_Contains
__global__ void contains_kernel(const int64_t* __restrict__ area_p, const int64_t* __restrict__ area_q, int64_t np,
                                int64_t nq, const int2* __restrict__ pairs, int64_t n,
                                const long long* __restrict__ inter, uint8_t* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int2 pq = pairs[k];
    uint8_t c = 0;
    if ((unsigned)pq.x < (unsigned long long)np && (unsigned)pq.y < (unsigned long long)nq) {
      const long long I = inter[k], ap = area_p[pq.x], aq = area_q[pq.y];
      // |p n q| == |q|: every pixel of q is a pixel of p
      c = (uint8_t)((I == aq && aq > 0 ? 1 : 0) | (I == ap && ap > 0 ? 2 : 0));
    }
    out[k] = c;
  }
}

static int blocks_for(int64_t n, int threads, int per_sm) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * per_sm;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

int run_contains(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
                 uint8_t* out, cudaStream_t stream) {
  contains_kernel<<<blocks_for(n, 256, 8), 256, 0, stream>>>(P->area, Q->area, P->n_polygons, Q->n_polygons,
                                                             reinterpret_cast<const int2*>(pairs), n,
                                                             reinterpret_cast<const long long*>(inter), out);
  return check_cuda(cudaGetLastError(), "sccg_contains");
}

// ------------------------------------------------------------- report
constexpr int kRepFields = (int)(sizeof(sccg_tile_report) / sizeof(long long));  // 15
static_assert(kRepFields == 15, "sccg_tile_report layout");
// field slots (sccg_sums layout, then the polygon counts)
enum { F_PAIRS = 0, F_NZ, F_I, F_U, F_AP, F_AQ, F_L0, F_L1, F_L2, F_L3, F_STATUS, F_NP, F_NQ, F_MP, F_MQ };

__device__ __forceinline__ int tile_of(const int4& m, const sccg_tiling& t) {
  // floor division of the (64-bit) offset from the grid origin, clamped into the grid
  const long long dx = (long long)m.x - t.x0, dy = (long long)m.y - t.y0;
  long long tx = dx >= 0 ? dx / t.tile_w : -((-dx + t.tile_w - 1) / t.tile_w);
  long long ty = dy >= 0 ? dy / t.tile_h : -((-dy + t.tile_h - 1) / t.tile_h);
  tx = tx < 0 ? 0 : (tx >= t.ntx ? t.ntx - 1 : tx);
  ty = ty < 0 ? 0 : (ty >= t.nty ? t.nty - 1 : ty);
  return (int)(ty * t.ntx + tx);
}

// One item per lane: a pair (k < n) or a polygon of P / Q.  Each lane carries
// its tile and its contribution to that tile's fields; the warp adds the
// contributions of lanes with the same tile (one group per distinct tile, a
// full-warp shuffle sum with the other lanes' values masked) and the group's
// first lane adds them into the tile with one atomic per non-zero field --
// integer adds, so the report is independent of the order.
__global__ void report_kernel(const int4* __restrict__ mbr_p, const int64_t* __restrict__ area_p, int64_t np,
                              const int4* __restrict__ mbr_q, const int64_t* __restrict__ area_q, int64_t nq,
                              const int2* __restrict__ pairs, int64_t n, const long long* __restrict__ inter,
                              const long long* __restrict__ uni, const unsigned* __restrict__ hit_p,
                              const unsigned* __restrict__ hit_q, sccg_tiling tl,
                              unsigned long long* __restrict__ tiles) {
  const int lane = threadIdx.x & 31;
  const int64_t total = n + np + nq;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < total; base += stride) {  // warp-uniform
    const int64_t i = base + lane;
    unsigned long long v[kRepFields];
#pragma unroll
    for (int f = 0; f < kRepFields; f++) v[f] = 0;
    int t = -1;
    if (i < n) {
      const int2 pq = pairs[i];
      if ((unsigned)pq.x < (unsigned long long)np && (unsigned)pq.y < (unsigned long long)nq) {
        t = tile_of(mbr_p[pq.x], tl);
        const long long I = inter[i], U = uni[i];
        v[F_PAIRS] = 1;
        v[F_I] = (unsigned long long)I;
        v[F_AP] = (unsigned long long)area_p[pq.x];
        v[F_AQ] = (unsigned long long)area_q[pq.y];
        if (I != 0) {  // Eq. (1) averages the pairs with |p n q| != 0
          v[F_NZ] = 1;
          v[F_U] = (unsigned long long)U;
          ratio_limbs(I, U, v[F_L0], v[F_L1], v[F_L2], v[F_L3]);
        }
      }
    } else if (i < n + np) {
      const int64_t p = i - n;
      t = tile_of(mbr_p[p], tl);
      v[F_NP] = 1;
      v[F_MP] = ((hit_p[p >> 5] >> (p & 31)) & 1u) ? 0 : 1;
    } else if (i < total) {
      const int64_t q = i - n - np;
      t = tile_of(mbr_q[q], tl);
      v[F_NQ] = 1;
      v[F_MQ] = ((hit_q[q >> 5] >> (q & 31)) & 1u) ? 0 : 1;
    }
    unsigned todo = __ballot_sync(FULL, t >= 0);
    while (todo) {  // warp-uniform: one round per distinct tile among the lanes
      const int leader = __ffs(todo) - 1;
      const int tt = __shfl_sync(FULL, t, leader);
      const bool mine = ((todo >> lane) & 1u) && t == tt;
      todo &= ~__ballot_sync(FULL, mine);
#pragma unroll
      for (int f = 0; f < kRepFields; f++) {
        const unsigned long long s = warp_sum_u64(mine ? v[f] : 0ull);
        if (lane == leader && s) atomicAdd(&tiles[(size_t)tt * kRepFields + f], s);
      }
    }
  }
}

int run_report(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
               const int64_t* uni, const uint32_t* hit_p, const uint32_t* hit_q, const sccg_tiling* tl,
               sccg_tile_report* tiles, cudaStream_t stream) {
  const int64_t total = n + P->n_polygons + Q->n_polygons;
  if (total == 0) return SCCG_OK;
  report_kernel<<<blocks_for(total, 256, 8), 256, 0, stream>>>(
      reinterpret_cast<const int4*>(P->mbr), P->area, P->n_polygons, reinterpret_cast<const int4*>(Q->mbr), Q->area,
      Q->n_polygons, reinterpret_cast<const int2*>(pairs), n, reinterpret_cast<const long long*>(inter),
      reinterpret_cast<const long long*>(uni), hit_p, hit_q, *tl, reinterpret_cast<unsigned long long*>(tiles));
  return check_cuda(cudaGetLastError(), "sccg_report");
}

// ------------------------------------------------- cross-rank reduction
constexpr int kSumsWords = (int)(sizeof(sccg_sums) / sizeof(long long));  // 11
constexpr int kAddWords = kSumsWords - 1;                                  // the additive fields
static_assert(SCCG_REDUCE_WORDS == kAddWords + 16, "reduce vector layout");

__global__ void sums_pack_kernel(const long long* __restrict__ s, long long* __restrict__ vec) {
  pdl_wait();
  const int i = threadIdx.x;
  if (i < kAddWords) vec[i] = s[i];
  else if (i < SCCG_REDUCE_WORDS) vec[i] = (s[kAddWords] >> (i - kAddWords)) & 1;
}

__global__ void sums_unpack_kernel(const long long* __restrict__ vec, long long* __restrict__ s) {
  pdl_wait();
  const int i = threadIdx.x;
  const unsigned bits = __ballot_sync(FULL, i >= kAddWords && i < SCCG_REDUCE_WORDS && vec[i] != 0);
  if (i < kAddWords) s[i] = vec[i];
  if (i == kAddWords) s[kAddWords] = (long long)(bits >> kAddWords);
}

cudaError_t launch_sums_pack(const sccg_sums* src, int64_t* vec, cudaStream_t st) {
  return launch_pdl(sums_pack_kernel, dim3(1), dim3(32), 0, st, reinterpret_cast<const long long*>(src),
                    reinterpret_cast<long long*>(vec));
}
cudaError_t launch_sums_unpack(const int64_t* vec, sccg_sums* dst, cudaStream_t st) {
  return launch_pdl(sums_unpack_kernel, dim3(1), dim3(32), 0, st, reinterpret_cast<const long long*>(vec),
                    reinterpret_cast<long long*>(dst));
}

}  // namespace sccg
