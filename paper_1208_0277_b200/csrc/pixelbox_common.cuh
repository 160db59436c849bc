// pixelbox_common.cuh -- pieces shared by the small-pair and the large-pair
// PixelBox kernels (pixelbox.cu, large.cu).  Not part of the ABI.
#pragma once
#include "internal.cuh"

namespace sccg {

constexpr unsigned FULL = 0xffffffffu;

struct Split {
  int kx, lkx, lsx, lsy, ncols, nrows;
  unsigned colpat;  // bit r*kx for every row r
};

__device__ __forceinline__ int ceil_log2(int v) { return v <= 1 ? 0 : 32 - __clz(v - 1); }

// SUBSAMPBOX (Alg. 1 l.30, reading R8): an aligned grid of power-of-two cells,
// 8 x 4 (or 4 x 8 for tall boxes), clipped to the box; every sub-box non-empty.
__device__ __forceinline__ Split make_split(int Wb, int Hb) {
  Split g;
  g.kx = Wb >= Hb ? 8 : 4;
  g.lkx = Wb >= Hb ? 3 : 2;
  const int ky = 32 / g.kx;
  g.lsx = ceil_log2((Wb + g.kx - 1) / g.kx);
  g.lsy = ceil_log2((Hb + ky - 1) / ky);
  g.ncols = (Wb + (1 << g.lsx) - 1) >> g.lsx;
  g.nrows = (Hb + (1 << g.lsy) - 1) >> g.lsy;
  g.colpat = g.kx == 8 ? 0x01010101u : 0x11111111u;
  return g;
}

// bits of sub-box rows r_lo..r_hi (empty if r_hi < r_lo)
__device__ __forceinline__ unsigned row_range(int r_lo, int r_hi, const Split& g) {
  return low_bits((r_hi - r_lo + 1) << g.lkx) << (max(r_lo, 0) << g.lkx);
}

// r = RN64(I / U) as an exact integer count of 2^-116, split into 30-bit limbs
// (reading R12).  Requires 0 < I <= U < 2^63.
__device__ __forceinline__ void ratio_limbs(long long I, long long U, unsigned long long& l0, unsigned long long& l1,
                                            unsigned long long& l2, unsigned long long& l3) {
  const double r = __ddiv_rn((double)I, (double)U);
  const unsigned long long bits = (unsigned long long)__double_as_longlong(r);
  const int ex = (int)((bits >> 52) & 0x7ff);
  const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
  const int s = ex - 1075 + 116;  // in [1, 64] for r in (2^-63, 1]
  const unsigned __int128 v = (unsigned __int128)mant << s;
  l0 = (unsigned long long)(v & 0x3fffffffu);
  l1 = (unsigned long long)((v >> 30) & 0x3fffffffu);
  l2 = (unsigned long long)((v >> 60) & 0x3fffffffu);
  l3 = (unsigned long long)(v >> 90);
}

// r = RN64(I / U) as an exact integer count of 2^-116, split into 30-bit limbs
// (reading R12), accumulated.  Requires 0 < I <= U < 2^63.
__device__ __forceinline__ void add_ratio_limbs(long long I, long long U, unsigned long long limb[4]) {
  unsigned long long a, b, c, d;
  ratio_limbs(I, U, a, b, c, d);
  limb[0] += a;
  limb[1] += b;
  limb[2] += c;
  limb[3] += d;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// --------------------------------------------------------------- large pairs
// Generic warp-per-pair kernel: any box size, sampling boxes + pixelization,
// shared-memory overflow path.  Consumes the pair indices the small-pair
// kernel routed to it (list[0 .. *count)).
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// PixelBox over the pairs the small kernel routed to the large path
// (large.cu): region work items with local edge culling.
int launch_large(const DevSet& Ps, const DevSet& Qs, const int2* pairs, long long n_cap, const long long* large_list,
                 const unsigned* large_count, long long* inter, long long* uni, sccg_sums* sums, int T, int mode,
                 long long* counters, void* ws, size_t ws_bytes, cudaStream_t stream);
size_t large_ws_bytes(long long n_cap);

}  // namespace sccg
