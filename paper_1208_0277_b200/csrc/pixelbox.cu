// pixelbox.cu -- the PixelBox kernel for small pairs
// and the sccg_pixelbox launcher.
//
// PAPER.md §3 / Algorithm 1 computes, per polygon pair, the area
// of intersection by recursively partitioning the pair's box into sampling
// boxes (§3.2), classifying each against both polygons as inside /
// outside / hover (Lemma 1), and pixelizing boxes smaller than a
// threshold T (Alg. 1 l.22) by ray-casting crossing counts (§3.1).
// The union follows from |p u q| = |p| + |q| - |p n q|.
//
// B200 design: the common nucleus pair (root box at most
// 32 x 32 and below T, so Alg. 1 pixelizes the root box directly) runs in the
// software-pipelined small kernel below -- one warp per pair, bit-parallel
// pixelization (a lane owns a 32-pixel row word; one crossing test decides 32
// ray casts).  Every other pair is routed to the large-pair path (large.cu):
// region work items, each a warp-private sampling-box DFS over locally culled
// edges.  Areas are exact integers; per-pair results and the int64 sums are
// bit-identical for every launch shape and threshold.
#include "pixelbox_common.cuh"

namespace sccg {

// --------------------------------------------------------------- small pairs
// The common case (nucleus pairs): root box at most 32 x 32 pixels and below
// T, each polygon at most kSmallCap vertical edges.  A warp claims 32 pairs,
// loads their metadata lane-parallel (32 independent loads in flight), then
// walks them with a software pipeline: while pair j is pixelized, pair j+1's
// edge records are already in flight into registers.  Pixelization is one row
// per lane (one 32-bit row word), half-warp per polygon when the box has at
// most 16 rows.  Per-pair results and sums are written lane-parallel.
constexpr int kSmallWarps = 8;
constexpr int kSmallCap = 128;   // vertical edges per polygon on this path (> 64: the non-pipelined loop)
constexpr int kPipeCap = 64;     // ... on the pipelined loop (two records per lane in registers)
constexpr int kSmallQOff = 136;  // q buffer offset in records (8 B): 1088 B, so p[t] and q[t] hit different banks

// Stage one polygon's row-crossing edges for a box of H <= 32 rows and
// W <= 32 columns as {row bits, pixel mask}: bit r of `rows` is set iff the
// edge crosses row r of the box (ylo <= r < yhi), `mask` holds the pixels the
// edge toggles.  Edges crossing no row are culled; every slot of the 32-record
// block (64 with `two`) is written -- kept records first, then zero records
// (no-ops) -- so no padding pass is needed.  Returns the loop length.
__device__ __forceinline__ int stage_rows(uint64_t r0, uint64_t r1, int nv, bool two, unsigned o0, int dx, int dy,
                                          int H, int2* buf) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  int c, lo, hi;
  decode_edge(r0, o0, c, lo, hi);
  unsigned rows = low_bits(min(hi + dy, H)) & ~low_bits(lo + dy);
  bool keep = lane < nv && rows != 0;
  unsigned b = __ballot_sync(FULL, keep);
  int cnt = __popc(b);
  buf[keep ? __popc(b & lt) : cnt + __popc(~b & lt)] =
      keep ? make_int2((int)rows, (int)suffix_mask(c + dx)) : make_int2(0, 0);
  if (!two) return cnt;
  decode_edge(r1, o0, c, lo, hi);
  rows = low_bits(min(hi + dy, H)) & ~low_bits(lo + dy);
  keep = lane + 32 < nv && rows != 0;
  b = __ballot_sync(FULL, keep);
  cnt = __popc(b);
  buf[32 + (keep ? __popc(b & lt) : cnt + __popc(~b & lt))] =
      keep ? make_int2((int)rows, (int)suffix_mask(c + dx)) : make_int2(0, 0);
  return 32 + cnt;
}

// stage_rows for up to 4 blocks of 32 records read from `rec` (L1-resident
// after the first window); returns 32 (nb - 1) + the last block's kept count.
__device__ __forceinline__ int stage_blocks(const uint64_t* __restrict__ rec, int nv, int nb, unsigned o0, int dx,
                                            int dy, int H, int2* buf) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  int cnt = 0;
#pragma unroll
  for (int blk = 0; blk < 4; blk++) {
    if (blk < nb) {
      int c, lo, hi;
      decode_edge(lane + 32 * blk < nv ? __ldg(rec + 32 * blk + lane) : 0ull, o0, c, lo, hi);
      const unsigned rows = low_bits(min(hi + dy, H)) & ~low_bits(lo + dy);
      const bool keep = lane + 32 * blk < nv && rows != 0;
      const unsigned b = __ballot_sync(FULL, keep);
      cnt = __popc(b);
      buf[32 * blk + (keep ? __popc(b & lt) : cnt + __popc(~b & lt))] =
          keep ? make_int2((int)rows, (int)suffix_mask(c + dx)) : make_int2(0, 0);
    }
  }
  return 32 * (nb - 1) + cnt;
}

// m ^= mask if (rows & bit) != 0 -- one predicate-producing LOP3 and one
// predicated LOP3 (the crossing test of one row against one edge).
__device__ __forceinline__ void xor_if(unsigned& m, unsigned rows, unsigned bit, unsigned mask) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.b32 p, t, 0;\n\t@p xor.b32 %0, %0, %3;\n\t}"
      : "+r"(m)
      : "r"(rows), "r"(bit), "r"(mask));
}

// Crossing parity words of rows `bit0` (and `bit1` when TWO) over n staged
// edges (n a multiple of 4; two records per 16-byte shared load).
template <bool TWO>
__device__ __forceinline__ void row_words(const int2* __restrict__ b, int n, unsigned bit0, unsigned bit1,
                                          unsigned& m0, unsigned& m1) {
  const int4* b4 = reinterpret_cast<const int4*>(b);
  for (int t = 0; t < (n >> 1); t += 2) {
    const int4 u = b4[t], w = b4[t + 1];
    xor_if(m0, u.x, bit0, u.y);
    xor_if(m0, u.z, bit0, u.w);
    xor_if(m0, w.x, bit0, w.y);
    xor_if(m0, w.z, bit0, w.w);
    if (TWO) {
      xor_if(m1, u.x, bit1, u.y);
      xor_if(m1, u.z, bit1, u.w);
      xor_if(m1, w.x, bit1, w.y);
      xor_if(m1, w.z, bit1, w.w);
    }
  }
}

#ifndef SCCG_SMALL_MINB
#define SCCG_SMALL_MINB 4
#endif
template <bool COUNT>
__global__ void __launch_bounds__(kSmallWarps * 32, SCCG_SMALL_MINB)
    small_kernel(DevSet Ps, DevSet Qs, const int2* __restrict__ pairs, long long n_cap,
                 const long long* __restrict__ dev_result, long long* __restrict__ inter,
                 long long* __restrict__ uni, sccg_sums* sums, int T, int mode, bool use_raster,
                 unsigned long long* queue,
                 LargeWs lw, long long* counters, unsigned* __restrict__ hit_p, unsigned* __restrict__ hit_q,
                 long long np_,
                 long long nq_) {
  pdl_entry_deferred();
  // pair count: host-given, or (async path) the filter's device-side count clamped to the buffer
  // (a join that overflowed the buffer left it incomplete: nothing is processed, the status says so)
  const long long r0 = dev_result ? ld_coherent(dev_result) : 0;
  const bool overflow = dev_result && r0 > n_cap;
  const long long n = dev_result ? (overflow ? 0 : r0) : n_cap;
  if (dev_result && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long r1 = ld_coherent(dev_result + 1);
    if (r1 || overflow)
      atomicOr(reinterpret_cast<unsigned long long*>(&sums->status),
               (unsigned long long)r1 | (overflow ? (unsigned long long)SCCG_STATUS_CAPACITY : 0ull));
  }
  __shared__ __align__(16) int2 s_buf[kSmallWarps][2 * kSmallQOff];
  __shared__ int4 s_meta[kSmallWarps][32];
  __shared__ int2 s_ep[kSmallWarps][32];
  __shared__ uint2 s_o0[kSmallWarps][32];  // the pair's record rebases (ecount.y of p and q)
  __shared__ unsigned long long s_acc[kSmallWarps][16];
  __shared__ int s_rstart[kSmallWarps][33];  // raster pairs: first (pair, row) item of each pair
  __shared__ unsigned s_rcnt[kSmallWarps][32];
  __shared__ const unsigned* s_rp[kSmallWarps][32];  // raster row of box row 0, per pair (p and q)
  __shared__ const unsigned* s_rq[kSmallWarps][32];
  __shared__ unsigned s_rsh[kSmallWarps][32];        // column shifts (p, q) and box width
  __shared__ unsigned char s_rmap[kSmallWarps][1024]; // item -> pair
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int2* bp = s_buf[warp];
  int2* bq = bp + kSmallQOff;
  int4* meta = s_meta[warp];
  int2* epq = s_ep[warp];
  if (lane == 0)
    for (int i = 0; i < 16; i++) s_acc[warp][i] = 0;
  unsigned status = 0;
  for (;;) {
    unsigned long long k0 = 0;
    if (lane == 0) k0 = atomicAdd(queue, 32ull);
    k0 = __shfl_sync(FULL, k0, 0);
    if ((long long)k0 >= n) break;
    const long long k = (long long)k0 + lane;
    // ---- lane-parallel metadata of pair k0 + lane
    bool ok = false, small = false, empty = false;
    int2 pq = make_int2(0, 0);
    int W = 0, H = 0;
    unsigned rast = 0u;
    if (k < n) {
      pq = pairs[k];
      ok = (unsigned)pq.x < (unsigned long long)np_ && (unsigned)pq.y < (unsigned long long)nq_;
      if (!ok) status |= SCCG_STATUS_ARG;  // index out of range: pair skipped
    }
    if (ok) {
      const int4 mp = Ps.mbr[pq.x], mq = Qs.mbr[pq.y];
      const int2 cpr = Ps.ecount[pq.x], cqr = Qs.ecount[pq.y];
      const int2 cp = make_int2(cpr.x & kNvMask, cpr.y), cq = make_int2(cqr.x & kNvMask, cqr.y);
      const long long op = Ps.off[pq.x], oq = Qs.off[pq.y];
      const int bx0 = max(mp.x, mq.x), by0 = max(mp.y, mq.y);
      W = min(mp.z, mq.z) - bx0;
      H = min(mp.w, mq.w) - by0;
      const int dxp = mp.x - bx0, dyp = mp.y - by0, dxq = mq.x - bx0, dyq = mq.y - by0;
      empty = !(W > 0 && H > 0);  // reading R18: I = 0
      small = mode == 0 && !empty && W <= 64 && H <= 64 && W * H < T && cp.x <= kSmallCap && cq.x <= kSmallCap &&
              op + cp.x < (1ll << 31) && oq + cq.x < (1ll << 31) && min(min(dxp, dyp), min(dxq, dyq)) >= -32768;
      if (mode != 0) {  // PixelOnly / NoSep (§5.2 baselines): the box of MBR(p) u MBR(q), union counted directly
        empty = false;
        W = max(mp.z, mq.z) - min(mp.x, mq.x);
        H = max(mp.w, mq.w) - min(mp.y, mq.y);
      }
      // both rings carry a raster (prep): the pair reads pixel classifications instead of edges.
      // meta.x: W (bits 0-6), H (7-13), nv_p (14-21), nv_q (22-29), raster (30)
      rast = (small && use_raster && W <= 32 && H <= 32 && (cpr.x & kRasterFlag) && (cqr.x & kRasterFlag)) ? 1u : 0u;
      meta[lane] = make_int4((int)((unsigned)W | ((unsigned)H << 7) | ((unsigned)cp.x << 14) | ((unsigned)cq.x << 22) |
                                   (rast << 30)),
                             (int)(((unsigned)dxp & 0xffffu) | ((unsigned)dyp << 16)),
                             (int)(((unsigned)dxq & 0xffffu) | ((unsigned)dyq << 16)), 0);
      epq[lane] = make_int2((int)op, (int)oq);
      s_o0[warp][lane] = make_uint2((unsigned)cp.y, (unsigned)cq.y);
    }
    __syncwarp();
    // ---- everything else goes to the generic kernel (warp-aggregated append)
    const bool large = ok && !empty && !small;
    const unsigned lb = __ballot_sync(FULL, large);
    if (lb) {
      unsigned base = 0;
      if (lane == 0) base = (unsigned)atomicAdd(&lw.ctr[2], (unsigned long long)__popc(lb));
      base = __shfl_sync(FULL, base, 0);
      if (large) emit_large(lw, base + __popc(lb & lanemask_lt()), k, W, H);
    }
    // ---- small pairs, software-pipelined: records of the next pair are in
    // flight into registers while the current pair is pixelized
    unsigned myI = 0;
    // ---- raster pairs, batched: the chunk's (pair, two rows) items are spread
    // over the lanes, so each lane has many independent row loads in flight; a
    // row costs two loads, two shifts, an AND and a popcount (memoized
    // pixelization)
    const unsigned rmask = __ballot_sync(FULL, rast != 0u);
    if (rmask) {
      const int hl = rast ? (H + 1) >> 1 : 0;  // items: row pairs
      int sc = hl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, sc, o);
        if (lane >= o) sc += t;
      }
      const int R = __shfl_sync(FULL, sc, 31);
      int* rstart = s_rstart[warp];
      unsigned* rcnt = s_rcnt[warp];
      unsigned char* rmap = s_rmap[warp];
      rstart[lane] = sc - hl;
      rcnt[lane] = 0u;
      if (rast) {
        const int4 mm = meta[lane];
        const int2 e = epq[lane];
        const unsigned mj = (unsigned)mm.x;
        s_rp[warp][lane] = reinterpret_cast<const unsigned*>(Ps.edges + e.x + ((mj >> 14) & 255)) - (mm.y >> 16);
        s_rq[warp][lane] = reinterpret_cast<const unsigned*>(Qs.edges + e.y + ((mj >> 22) & 255)) - (mm.z >> 16);
        s_rsh[warp][lane] = (unsigned)(-(int)(short)(mm.y & 0xffff)) | ((unsigned)(-(int)(short)(mm.z & 0xffff)) << 8) |
                            ((unsigned)W << 16) | ((unsigned)H << 24);
      }
      // item -> pair map: each lane writes its own pair's run (a loop of
      // max(hl) <= 16 byte stores; a pair-by-pair cooperative loop over the
      // ~32 raster pairs cost ~30 % of the kernel's instructions, profiles/r01)
      for (int i = 0, st = sc - hl; i < hl; i++) rmap[st + i] = (unsigned char)lane;
      __syncwarp();
      const unsigned le = lanemask_lt() | (1u << lane);
      // kU 32-item groups per round: all row loads are issued before any is
      // consumed (many loads in flight per lane)
#ifndef SCCG_RASTER_GROUPS
#define SCCG_RASTER_GROUPS 3  // row-load groups in flight per lane (measured: 3 < 2 < 4 < 6 in time)
#endif
      constexpr int kU = SCCG_RASTER_GROUPS;
      for (int t0 = 0; t0 < R; t0 += 32 * kU) {  // warp-uniform trip count
        unsigned wpv[kU], wqv[kU], wpw[kU], wqw[kU], shv[kU];
        int jrv[kU];
        bool hv[kU], av[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const int t = t0 + 32 * u + lane;
          av[u] = t < R;
          hv[u] = !av[u] || lane == 0;
          jrv[u] = 0;
          wpv[u] = wqv[u] = wpw[u] = wqw[u] = shv[u] = 0u;
          if (av[u]) {
            const int jr = rmap[t];
            const int i = t - rstart[jr], r = 2 * i;
            hv[u] |= i == 0;
            jrv[u] = jr;
            const unsigned sh = s_rsh[warp][jr];
            shv[u] = sh;
            const unsigned* rp = s_rp[warp][jr] + r;
            const unsigned* rq = s_rq[warp][jr] + r;
            wpv[u] = __ldg(rp);
            wqv[u] = __ldg(rq);
            if (r + 1 < (int)(sh >> 24)) {  // an odd box height leaves the last item one row
              wpw[u] = __ldg(rp + 1);
              wqw[u] = __ldg(rq + 1);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
          if (t0 + 32 * u >= R) break;  // warp-uniform
          const unsigned sh = shv[u];
          const unsigned sp = sh & 0xffu, sq = (sh >> 8) & 0xffu, wm = low_bits((int)((sh >> 16) & 0xffu));
          unsigned c = av[u] ? (unsigned)(__popc((wpv[u] >> sp) & (wqv[u] >> sq) & wm) +
                                          __popc((wpw[u] >> sp) & (wqw[u] >> sq) & wm))
                             : 0u;
          // each pair's items occupy consecutive lanes: segmented shuffle sum,
          // the segment's first lane adds it to the pair's count
          const unsigned heads = __ballot_sync(FULL, hv[u]);
          const unsigned after = heads & ~le;
          const int next = after ? __ffs(after) - 1 : 32;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_down_sync(FULL, c, o);
            if (lane + o < next) c += v;
          }
          if (av[u] && ((heads >> lane) & 1u)) rcnt[jrv[u]] += c;
          __syncwarp();
        }
      }
      __syncwarp();
      if (rast) myI = rcnt[lane];
    }
    const unsigned wide = __ballot_sync(FULL, small && max(((unsigned)meta[lane].x >> 14) & 255,
                                                             ((unsigned)meta[lane].x >> 22) & 255) > kPipeCap);
    unsigned todo = __ballot_sync(FULL, small) & ~rmask & ~wide;
    uint64_t np0 = 0, np1 = 0, nq0 = 0, nq1 = 0;
    auto prefetch = [&](int j) {
      const int4 mm = meta[j];
      const unsigned mj = (unsigned)mm.x;
      const int2 e = epq[j];
      const int nvp = (mj >> 14) & 255, nvq = (mj >> 22) & 255;
      const uint64_t* pe = Ps.edges + e.x;
      const uint64_t* qe = Qs.edges + e.y;
      np0 = lane < nvp ? __ldg(pe + lane) : 0ull;
      nq0 = lane < nvq ? __ldg(qe + lane) : 0ull;
      if (nvp > 32) np1 = lane + 32 < nvp ? __ldg(pe + 32 + lane) : 0ull;
      if (nvq > 32) nq1 = lane + 32 < nvq ? __ldg(qe + 32 + lane) : 0ull;
    };
    if (todo) prefetch(__ffs(todo) - 1);
    unsigned long long c_tests = 0;
    const unsigned bit0 = 1u << (lane & 15), bit1 = 1u << ((lane & 15) + 16);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t cp0 = np0, cp1 = np1, cq0 = nq0, cq1 = nq1;
      if (todo) prefetch(__ffs(todo) - 1);
      const int4 mm = meta[j];
      const unsigned mj = (unsigned)mm.x, dpj = (unsigned)mm.y, dqj = (unsigned)mm.z;
      const int Wb = mj & 127, Hb = (mj >> 7) & 127, nvp = (mj >> 14) & 255, nvq = (mj >> 22) & 255;
      const bool two = max(nvp, nvq) > 32;
      const int dxp = (int)(short)(dpj & 0xffffu), dyp = (int)dpj >> 16;
      const int dxq = (int)(short)(dqj & 0xffffu), dyq = (int)dqj >> 16;
      // boxes up to 64 x 64 in windows of <= 32 x 32: the records stay in
      // registers; a record left of a window toggles all of its pixels
      unsigned Ij = 0;
      for (int wy = 0; wy < Hb; wy += 32)
        for (int wx = 0; wx < Wb; wx += 32) {
          const int W = min(32, Wb - wx), H = min(32, Hb - wy);
          const uint2 rb = s_o0[warp][j];
          const int cntp = stage_rows(cp0, cp1, nvp, two, rb.x, dxp - wx, dyp - wy, H, bp);
          const int cntq = stage_rows(cq0, cq1, nvq, two, rb.y, dxq - wx, dyq - wy, H, bq);
          // half-warp per polygon (lanes 0-15: p, 16-31: q), rows lane&15 (+16)
          const int npad = (max(cntp, cntq) + 3) & ~3;
          __syncwarp();
          const int2* b = lane < 16 ? bp : bq;
          unsigned m0 = 0, m1 = 0;
          if (H <= 16)
            row_words<false>(b, npad, bit0, bit1, m0, m1);
          else
            row_words<true>(b, npad, bit0, bit1, m0, m1);
          const unsigned o0 = __shfl_xor_sync(FULL, m0, 16), o1 = __shfl_xor_sync(FULL, m1, 16);
          const unsigned wmask = low_bits(W);
          const unsigned cnt = lane < 16 ? __popc(m0 & o0 & wmask) + __popc(m1 & o1 & wmask) : 0u;
          Ij += __reduce_add_sync(FULL, cnt);
          if (COUNT) c_tests += (unsigned long long)H * (cntp + cntq);
          __syncwarp();  // buffers are rewritten by the next window / pair
        }
      if (lane == j) myI = Ij;
    }
    // ---- small pairs with more than kPipeCap edges in a polygon: records
    // loaded straight into registers (up to 4 per lane), not pipelined
    for (unsigned wd = wide; wd; wd &= wd - 1) {
      const int j = __ffs(wd) - 1;
      const int4 mm = meta[j];
      const unsigned mj = (unsigned)mm.x, dpj = (unsigned)mm.y, dqj = (unsigned)mm.z;
      const int Wb = mj & 127, Hb = (mj >> 7) & 127, nvp = (mj >> 14) & 255, nvq = (mj >> 22) & 255;
      const int nb = (max(nvp, nvq) + 31) >> 5;
      const int2 e = epq[j];
      const uint64_t* rp = Ps.edges + e.x;
      const uint64_t* rq = Qs.edges + e.y;
      const int dxp = (int)(short)(dpj & 0xffffu), dyp = (int)dpj >> 16;
      const int dxq = (int)(short)(dqj & 0xffffu), dyq = (int)dqj >> 16;
      unsigned Ij = 0;
      for (int wy = 0; wy < Hb; wy += 32)
        for (int wx = 0; wx < Wb; wx += 32) {
          const int W = min(32, Wb - wx), H = min(32, Hb - wy);
          const uint2 rb = s_o0[warp][j];
          const int cntp = stage_blocks(rp, nvp, nb, rb.x, dxp - wx, dyp - wy, H, bp);
          const int cntq = stage_blocks(rq, nvq, nb, rb.y, dxq - wx, dyq - wy, H, bq);
          const int npad = (max(cntp, cntq) + 3) & ~3;
          __syncwarp();
          const int2* b = lane < 16 ? bp : bq;
          unsigned m0 = 0, m1 = 0;
          if (H <= 16)
            row_words<false>(b, npad, bit0, bit1, m0, m1);
          else
            row_words<true>(b, npad, bit0, bit1, m0, m1);
          const unsigned o0 = __shfl_xor_sync(FULL, m0, 16), o1 = __shfl_xor_sync(FULL, m1, 16);
          const unsigned wmask = low_bits(W);
          const unsigned cnt = lane < 16 ? __popc(m0 & o0 & wmask) + __popc(m1 & o1 & wmask) : 0u;
          Ij += __reduce_add_sync(FULL, cnt);
          if (COUNT) c_tests += (unsigned long long)H * (cntp + cntq);
          __syncwarp();
        }
      if (lane == j) myI = Ij;
    }
    // ---- lane-parallel outputs and batch totals
    const unsigned long long c_px_all = COUNT ? warp_sum_u64(small ? (unsigned long long)W * H : 0ull) : 0ull;
    const bool done = ok && (small || empty);
    unsigned long long v_i = 0, v_u = 0, v_ap = 0, v_aq = 0, l0 = 0, l1 = 0, l2 = 0, l3 = 0;
    unsigned nz = 0;
    if (done) {
      const long long ap = Ps.area[pq.x], aq = Qs.area[pq.y];
      const long long I = small ? (long long)myI : 0;
      const long long U = ap + aq - I;  // indirect union
      if (inter) inter[k] = I;
      if (uni) uni[k] = U;
      v_i = I;
      v_ap = ap;
      v_aq = aq;
      if (I != 0) {
        nz = 1;
        v_u = U;
        if (hit_p) atomicOr(&hit_p[pq.x >> 5], 1u << (pq.x & 31));
        if (hit_q) atomicOr(&hit_q[pq.y >> 5], 1u << (pq.y & 31));
        ratio_limbs(I, U, l0, l1, l2, l3);
      }
    }
    const unsigned n_small = __popc(__ballot_sync(FULL, small));
    const unsigned n_done = __popc(__ballot_sync(FULL, done));
    const unsigned n_nz = __popc(__ballot_sync(FULL, nz != 0));
    v_i = __reduce_add_sync(FULL, (unsigned)v_i);  // <= 32 * 1024
    v_u = warp_sum_u64(v_u);
    v_ap = warp_sum_u64(v_ap);
    v_aq = warp_sum_u64(v_aq);
    l0 = warp_sum_u64(l0);
    l1 = warp_sum_u64(l1);
    l2 = warp_sum_u64(l2);
    l3 = warp_sum_u64(l3);
    if (lane == 0) {
      unsigned long long* a = s_acc[warp];
      a[0] += n_done;
      a[1] += n_nz;
      a[2] += v_i;
      a[3] += v_u;
      a[4] += v_ap;
      a[5] += v_aq;
      a[6] += l0;
      a[7] += l1;
      a[8] += l2;
      a[9] += l3;
      if (COUNT) {
        a[11] += c_tests;
        a[12] += c_px_all;
        a[13] += n_small;
      }
    }
  }
  pdl_done();  // the queue is drained: the item kernel may launch
  status = __reduce_or_sync(FULL, status);
  if (lane == 0) s_acc[warp][10] |= status;
  __syncthreads();
  if (threadIdx.x < 14) {
    unsigned long long v = 0;
    for (int w = 0; w < kSmallWarps; w++) v = threadIdx.x == 10 ? (v | s_acc[w][10]) : v + s_acc[w][threadIdx.x];
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(sums);
    if (threadIdx.x < 10) {
      if (v) atomicAdd(&dst[threadIdx.x], v);
    } else if (threadIdx.x == 10) {
      if (v) atomicOr(&dst[10], v);
    } else if (COUNT && v) {
      const int slot = threadIdx.x == 11 ? SCCG_CNT_ROWTESTS : threadIdx.x == 12 ? SCCG_CNT_PIXELS : SCCG_CNT_PIXBOXES;
      atomicAdd((unsigned long long*)&counters[slot], v);
      if (threadIdx.x == 12) atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROOTPX], v);
    }
  }
}

// ---------------------------------------------------------------------- host
struct PixelboxWs {
  unsigned long long* queue;  // small-kernel queue
  void* large;
  size_t large_bytes;
};

static size_t pixelbox_layout(int64_t n, Carve& cv, PixelboxWs& w) {
  w.queue = cv.take<unsigned long long>(4);
  w.large_bytes = large_ws_bytes(n);
  w.large = cv.take<char>(w.large_bytes);
  return cv.used;
}

size_t pixelbox_ws_bytes(int64_t n) {
  Carve cv{nullptr, ~size_t(0)};
  PixelboxWs w;
  return pixelbox_layout(n, cv, w) + 256;
}

__global__ void zero_counters_kernel(unsigned long long* queue, unsigned long long* ctr) {
  pdl_entry();  // the small kernel chains onto this one: its completion must imply the join's
  if (threadIdx.x < 4) queue[threadIdx.x] = 0ull;
  else if (threadIdx.x < 8) ctr[threadIdx.x - 4] = 0ull;
}

int run_pixelbox(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n,
                 const int64_t* dev_result, int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg,
                 void* ws, size_t ws_bytes, cudaStream_t stream) {
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  PixelboxWs w;
  pixelbox_layout(n, cv, w);
  if (!cv.ok || ws == nullptr) return set_error(SCCG_E_WORKSPACE, "pixelbox workspace too small");
  // workspace beyond the required part: the large path's edge-index pool (optional)
  const size_t used = (cv.used + 255) & ~size_t(255);
  void* pool = ws_bytes > used ? reinterpret_cast<char*>(ws) + used : nullptr;
  const size_t pool_bytes = ws_bytes > used ? ws_bytes - used : 0;
  int T = cfg && cfg->threshold > 0 ? cfg->threshold : 2048;
  const int mode = cfg ? cfg->mode : 0;
  const bool use_raster = !(cfg && (cfg->flags & SCCG_FLAG_NO_RASTER));
  if (T < 2) T = 2;
  if (mode < 0 || mode > 2) return set_error(SCCG_E_ARG, "config.mode must be 0 (PixelBox), 1 (PixelOnly) or 2 (NoSep)");
  bool lok = true;
  const LargeWs lw = large_ws(n, w.large, w.large_bytes, pool, pool_bytes, lok);
  if (!lok) return set_error(SCCG_E_WORKSPACE, "pixelbox (large) workspace too small");
  // the small kernel's queue and the large path's counters: one memset when
  // they are neighbours in the workspace (they are: pixelbox_layout)
  // (a one-warp kernel, so the small kernel chains onto it by PDL)
  launch_pdl(zero_counters_kernel, dim3(1), dim3(32), 0, stream, w.queue, lw.ctr);
  if (n == 0) return check_cuda(cudaGetLastError(), "pixelbox");
  const bool count = cfg && cfg->counters;
  long long* counters = count ? reinterpret_cast<long long*>(cfg->counters) : nullptr;
  static int sms = 0, per_sm_s[2] = {0, 0};
  if (sms == 0) {  // launch geometry, queried once
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s[1], small_kernel<true>, kSmallWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s[0], small_kernel<false>, kSmallWarps * 32, 0);
  }
  int64_t grid_s = cfg && cfg->grid > 0 ? cfg->grid : (int64_t)sms * max(per_sm_s[count], 1);
  const int64_t need = (n + kSmallWarps * 32 - 1) / (kSmallWarps * 32);
  if (grid_s > need) grid_s = need;
  if (grid_s < 1) grid_s = 1;
  DevSet Ps = dev_set(p), Qs = dev_set(q);
  const int2* pr = reinterpret_cast<const int2*>(pairs);
  long long* in = reinterpret_cast<long long*>(inter);
  long long* un = reinterpret_cast<long long*>(uni);
  const long long* dr = reinterpret_cast<const long long*>(dev_result);
  unsigned* hp = cfg ? reinterpret_cast<unsigned*>(cfg->hit_p) : nullptr;
  unsigned* hq = cfg ? reinterpret_cast<unsigned*>(cfg->hit_q) : nullptr;
  if (count)
    launch_pdl(small_kernel<true>, dim3((unsigned)grid_s), dim3(kSmallWarps * 32), 0, stream, Ps, Qs, pr, (long long)n,
               dr, in, un, sums, T, mode, use_raster, w.queue, lw, counters, hp, hq, (long long)p->n_polygons,
               (long long)q->n_polygons);
  else
    launch_pdl(small_kernel<false>, dim3((unsigned)grid_s), dim3(kSmallWarps * 32), 0, stream, Ps, Qs, pr,
               (long long)n, dr, in, un, sums, T, mode, use_raster, w.queue, lw, (long long*)nullptr, hp, hq,
               (long long)p->n_polygons, (long long)q->n_polygons);
  if (int r = check_cuda(cudaGetLastError(), "pixelbox small launch")) return r;
  const int dense = !(cfg && (cfg->flags & SCCG_FLAG_PAPER_SPLIT));
  return launch_large(Ps, Qs, pr, lw, in, un, sums, T, mode, dense, counters, hp, hq, stream);
}

}  // namespace sccg

namespace sccg {

__global__ void count_missing_kernel(const unsigned* __restrict__ hit, long long n, long long* out) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long c = 0;
  const long long nw = (n + 31) / 32;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (long long)gridDim.x * blockDim.x) {
    unsigned v = hit[i];
    if (i == nw - 1 && (n & 31)) v &= (1u << (n & 31)) - 1u;  // ignore bits past n
    c += (unsigned long long)__popc(v);
  }
  c = warp_sum_u64(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(out), s);
}

__global__ void set_kernel(long long* out, long long v) { *out = v; }

// sccg_sums_copy: 11 int64 by one warp; the fence makes host-memory
// destinations visible system-wide before the kernel completes
__global__ void sums_copy_kernel(const long long* __restrict__ src, volatile long long* dst) {
  pdl_wait();
  constexpr int kWords = (int)(sizeof(sccg_sums) / sizeof(long long));
  if (threadIdx.x < kWords) dst[threadIdx.x] = ld_coherent(src + threadIdx.x);  // written by atomics of the previous kernels
  __threadfence_system();
}

cudaError_t launch_sums_copy(const sccg_sums* src, sccg_sums* dst, cudaStream_t st) {
  return launch_pdl(sums_copy_kernel, dim3(1), dim3(32), 0, st, reinterpret_cast<const long long*>(src),
                    reinterpret_cast<volatile long long*>(dst));
}
__global__ void finish_missing_kernel(long long* out, long long n) { *out = n - *out; }

int count_missing(const uint32_t* hit, int64_t n, int64_t* out, cudaStream_t st) {
  // missing = n - (number of set bits): start at n, subtract via a negative add
  set_kernel<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(out), 0);
  if (n > 0) {
    const long long nw = (n + 31) / 32;
    const unsigned blocks = (unsigned)min((nw + 255) / 256, 1024ll);
    count_missing_kernel<<<blocks, 256, 0, st>>>(hit, n, reinterpret_cast<long long*>(out));
  }
  finish_missing_kernel<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(out), n);
  return check_cuda(cudaGetLastError(), "count missing");
}

}  // namespace sccg
