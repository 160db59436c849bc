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

// ---------------------------------------------------------- large-pair items
// A pair routed to the large path (large.cu) is cut into region work items
// (SURVEY §8 a3): its root box is split into nx x ny regions of about
// kRegion pixels per side.  Slot i of `items` (i = the pair's index in the
// large list) always holds region 0; the other regions are appended after
// n_cap.  rem[i] counts the pair's unfinished items; acc[i] accumulates its
// pixel count.
#ifndef SCCG_REGION
#define SCCG_REGION 128
#endif
constexpr int kRegion = SCCG_REGION;  // target region side
constexpr int kMaxSplit = 32;      // regions per axis at most
constexpr int kMaxRegion = 32766;  // local coordinates are 15-bit (plus clamp margin)

struct LargeWs {
  unsigned long long* ctr;  // [0] item queue, [1] extra item count, [2] large-pair count (low 32 bits),
                            // [3] words of the edge-index pool taken
  long long* list;          // [n_cap] pair index of large pair i
  long long* acc;           // [n_cap] |p n q| of large pair i
  long long* acc_u;         // [n_cap] |p u q| of large pair i (modes 1, 2: union counted directly)
  unsigned* rem;            // [n_cap] items of pair i not yet finished
  uint64_t* items;          // [n_cap + extra_cap]
  int* ixstate;             // [n_cap] edge index of pair i: 0 none yet, 2 ready, 3 not built (large.cu)
  long long* ixoff;         // [n_cap] its first pool word
  uint64_t* pool;           // the edge-index pool (workspace beyond sccg_pixelbox_workspace_bytes), or null
  long long pool_cap;       // its words
  long long n_cap, extra_cap;
};

// item: pair slot i (32 bit; 0xffffffff = no-op) | rx | ry | nx | ny (8 bit each)
__device__ __forceinline__ uint64_t pack_item(unsigned i, int rx, int ry, int nx, int ny) {
  return (uint64_t)i | ((uint64_t)rx << 32) | ((uint64_t)ry << 40) | ((uint64_t)nx << 48) | ((uint64_t)ny << 56);
}

// Register large pair i (pair index k, root box W x H) and its region items.
__device__ __forceinline__ void emit_large(const LargeWs& w, unsigned i, long long k, int W, int H) {
  int nx = min(kMaxSplit, max((W + kRegion - 1) / kRegion, (W + kMaxRegion - 1) / kMaxRegion));
  int ny = min(kMaxSplit, max((H + kRegion - 1) / kRegion, (H + kMaxRegion - 1) / kMaxRegion));
  w.list[i] = k;
  w.acc[i] = 0;
  w.acc_u[i] = 0;
  w.ixstate[i] = 0;
  const int extra = nx * ny - 1;
  if (extra > 0) {
    const long long base = (long long)atomicAdd(&w.ctr[1], (unsigned long long)extra);
    if (base + extra <= w.extra_cap) {
      for (int r = 1; r <= extra; r++) w.items[w.n_cap + base + r - 1] = pack_item(i, r % nx, r / nx, nx, ny);
    } else {  // out of item space: the pair is one item (split in-warp on overflow)
      for (long long t = base; t < w.extra_cap; t++) w.items[w.n_cap + t] = pack_item(0xffffffffu, 0, 0, 1, 1);
      nx = ny = 1;
    }
  }
  w.rem[i] = (unsigned)(nx * ny);
  w.items[i] = pack_item(i, 0, 0, nx, ny);
}

size_t large_ws_bytes(long long n_cap);
LargeWs large_ws(long long n_cap, void* ws, size_t ws_bytes, void* pool, size_t pool_bytes, bool& ok);
// the region-item kernel over everything the small kernel routed to the large path
int launch_large(const DevSet& Ps, const DevSet& Qs, const int2* pairs, const LargeWs& w, long long* inter,
                 long long* uni, sccg_sums* sums, int T, int mode, int dense, long long* counters, unsigned* hit_p,
                 unsigned* hit_q, cudaStream_t stream);

}  // namespace sccg
