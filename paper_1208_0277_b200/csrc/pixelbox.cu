// pixelbox.cu -- the PixelBox kernel for sm_100a.
//
// PAPER.md §3 / Algorithm 1 computes, per polygon pair, the area
// of intersection by recursively partitioning the pair's box into sampling
// boxes (§3.2), classifying each against both polygons as inside /
// outside / hover (Lemma 1), and pixelizing boxes smaller than a
// threshold T (Alg. 1 l.22) by ray-casting crossing counts (§3.1).
// The union follows from |p u q| = |p| + |q| - |p n q|.
//
// B200 design: one warp per pair, pairs pulled from a
// global work queue by a persistent grid; no __syncthreads in the pair loop
// (the paper's block-wide barrier per stack pop, and its read/write
// hazard, reading R11, disappear: the stack is warp-private and every pop is
// separated from the next push by __syncwarp).  Both phases are bit-parallel:
//   * pixelization: a lane owns a 32-pixel row word and accumulates the
//     crossing parity of all 32 pixels at once -- each vertical edge that
//     crosses the row toggles the pixels on one side of it (a shifted mask),
//     so one (row word x edge) test decides 32 ray casts;
//   * box classification (Lemma 1, reading R6-A): a box split into up to 32
//     power-of-two-aligned sub-boxes is classified edge-parallel -- a lane owns
//     an edge and writes the sub-boxes whose open interior the edge meets
//     (hover) and the sub-box corner pixels whose rays it crosses (parity) as
//     32-bit masks, OR / XOR-reduced across the warp with one REDUX each.
// Areas are exact integers; per-pair results and the int64 sums are
// bit-identical for every launch shape and threshold.
#include "internal.cuh"

namespace sccg {

constexpr int kWarps = 8;        // warps per CTA
constexpr int kStackCap = 512;   // sampling boxes per warp stack (>= 32 x depth)
constexpr int kECap = 128;       // staged vertical edges per polygon per warp
constexpr int kChunk = 4;        // pairs claimed per queue atomic
constexpr unsigned FULL = 0xffffffffu;

struct PairCtx {
  const uint64_t* ev;  // vertical edge records (sccg_prep)
  const int2* v;       // the ring's raw vertices (horizontal edges are read from these)
  int nv, nh, V;       // vertical edges, horizontal edges, vertices
  int dx, dy;          // polygon MBR origin minus root-box origin
  int ox, oy;          // root-box origin (absolute)
};

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

// Lemma 1 (reading R6-A) for all sub-boxes of one split, edge-parallel.
// hov: sub-boxes whose open interior meets a polygon edge; par: crossing
// parity of each sub-box's lower-left pixel (inside iff set), valid where
// hov == 0.  dx, dy: polygon MBR origin relative to the box origin.
__device__ __forceinline__ void classify(const PairCtx& c, int dx, int dy, int Wb, int Hb, const Split& g,
                                         unsigned& hov, unsigned& par) {
  const int lane = threadIdx.x & 31;
  const int sx = 1 << g.lsx, sy = 1 << g.lsy;
  unsigned h = 0, p = 0;
  for (int j = lane; j < c.nv; j += 32) {
    int cc, lo, hi;
    unpack_edge(__ldg(c.ev + j), cc, lo, hi);
    const int x = cc + dx, yl = lo + dy, yh = hi + dy;
    if (yl < Hb && yh > 0) {
      const int r_hi = min(g.nrows - 1, (yh - 1) >> g.lsy);
      if (x > 0 && x < Wb && (x & (sx - 1)) != 0)  // edge inside a column's open x-range
        h |= (g.colpat << (x >> g.lsx)) & row_range(max(0, yl >> g.lsy), r_hi, g);
      if (x > 0) {  // ray from corner pixel (c*sx, r*sy) crosses x iff c*sx < x and yl <= r*sy < yh
        const int c_hi = min(g.ncols - 1, (x - 1) >> g.lsx);
        p ^= (low_bits(c_hi + 1) * g.colpat) & row_range(max(0, (yl + sy - 1) >> g.lsy), r_hi, g);
      }
    }
  }
  // horizontal edges straight from the ring: edge (v_j, v_j+1) with equal y
  const int ax0 = c.ox + (c.dx - dx), ay0 = c.oy + (c.dy - dy);  // absolute origin of the box
  for (int j = lane; j < c.V; j += 32) {
    const int2 a = __ldg(c.v + j), b = __ldg(c.v + (j + 1 == c.V ? 0 : j + 1));
    if (a.y != b.y || a.x == b.x) continue;
    const int y = a.y - ay0, xl = min(a.x, b.x) - ax0, xh = max(a.x, b.x) - ax0;
    if (y > 0 && y < Hb && (y & (sy - 1)) != 0 && xl < Wb && xh > 0) {
      const int c_lo = max(0, xl >> g.lsx), c_hi = min(g.ncols - 1, (xh - 1) >> g.lsx);
      h |= low_bits(c_hi - c_lo + 1) << (((y >> g.lsy) << g.lkx) + c_lo);
    }
  }
  hov = __reduce_or_sync(FULL, h);
  par = __reduce_xor_sync(FULL, p);
}

// Stage the vertical edges of one polygon that cross any row of the box into
// shared memory as {ylo, span, mask | x, 0}, box-relative.  Returns the count
// (> kECap means the caller must stream edges from global memory instead).
__device__ __forceinline__ int stage(const PairCtx& c, int dx, int dy, int Hb, bool one_word, int4* buf) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int j0 = 0; j0 < c.nv; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    int x = 0, yl = 0, yh = 0;
    if (j < c.nv) {
      int cc, lo, hi;
      unpack_edge(__ldg(c.ev + j), cc, lo, hi);
      x = cc + dx;
      yl = lo + dy;
      yh = hi + dy;
      keep = yl < Hb && yh > 0;
    }
    const unsigned b = __ballot_sync(FULL, keep);
    if (keep) {
      const int pos = cnt + __popc(b & lanemask_lt());
      if (pos < kECap) buf[pos] = make_int4(yl, yh - yl, one_word ? (int)suffix_mask(x) : x, 0);
    }
    cnt += __popc(b);
  }
  return cnt;
}

// Row-word crossing parity from staged edges.
__device__ __forceinline__ unsigned row_parity_staged(const int4* buf, int n, int row, bool one_word, int xs) {
  unsigned m = 0;
  if (one_word) {
#pragma unroll 4
    for (int j = 0; j < n; j++) {
      const int4 r = buf[j];
      if ((unsigned)(row - r.x) < (unsigned)r.y) m ^= (unsigned)r.z;
    }
  } else {
#pragma unroll 4
    for (int j = 0; j < n; j++) {
      const int4 r = buf[j];
      if ((unsigned)(row - r.x) < (unsigned)r.y) m ^= suffix_mask(r.z - xs);
    }
  }
  return m;
}

// Row-word crossing parity streaming every vertical edge from global memory
// (shared-memory overflow path).
__device__ __forceinline__ unsigned row_parity_global(const PairCtx& c, int dx, int dy, int row, int xs) {
  unsigned m = 0;
  for (int j = 0; j < c.nv; j++) {
    int cc, lo, hi;
    unpack_edge(__ldg(c.ev + j), cc, lo, hi);
    if ((unsigned)(row - (lo + dy)) < (unsigned)(hi - lo)) m ^= suffix_mask(cc + dx - xs);
  }
  return m;
}

// Pixelization of box [X0, X1) x [Y0, Y1) (root-relative), Alg. 1 l.22-28:
// returns this lane's share of the pixels inside both polygons.
template <bool COUNT>
__device__ long long pixelize(int X0, int Y0, int X1, int Y1, const PairCtx& P, const PairCtx& Q, int4* sp,
                              int4* sq, long long* counters) {
  const int lane = threadIdx.x & 31;
  const int Wb = X1 - X0, Hb = Y1 - Y0;
  const int nw = (Wb + 31) >> 5;
  const bool one = nw == 1;
  const int dxp = P.dx - X0, dyp = P.dy - Y0, dxq = Q.dx - X0, dyq = Q.dy - Y0;
  const int np = stage(P, dxp, dyp, Hb, one, sp);
  const int nq = stage(Q, dxq, dyq, Hb, one, sq);
  __syncwarp();
  const bool over_p = np > kECap, over_q = nq > kECap;
  const int nseg = Hb * nw;
  long long acc = 0;
  for (int s0 = 0; s0 < nseg; s0 += 32) {
    const int s = s0 + lane;
    if (s < nseg) {
      const int row = one ? s : s / nw;
      const int xs = (s - row * nw) << 5;
      const unsigned mp = over_p ? row_parity_global(P, dxp, dyp, row, xs) : row_parity_staged(sp, np, row, one, xs);
      const unsigned mq = over_q ? row_parity_global(Q, dxq, dyq, row, xs) : row_parity_staged(sq, nq, row, one, xs);
      acc += __popc(mp & mq & low_bits(Wb - xs));
    }
  }
  __syncwarp();
  if (COUNT && lane == 0) {
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXELS], (unsigned long long)Wb * Hb);
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROWTESTS],
              (unsigned long long)nseg * ((over_p ? P.nv : np) + (over_q ? Q.nv : nq)));
    atomicAdd((unsigned long long*)&counters[SCCG_CNT_PIXBOXES], 1ull);
  }
  return acc;
}

__device__ __forceinline__ uint64_t pack_box(int x0, int y0, int x1, int y1) {
  return (uint64_t)(uint32_t)x0 | ((uint64_t)(uint32_t)y0 << 16) | ((uint64_t)(uint32_t)x1 << 32) |
         ((uint64_t)(uint32_t)y1 << 48);
}

// Sampling-box loop (Alg. 1 l.13-42) over a warp-private DFS stack.
template <bool COUNT>
__device__ long long sample(int W, int H, const PairCtx& P, const PairCtx& Q, uint64_t* stk, int4* sp, int4* sq, int T,
                            long long* counters, unsigned& status) {
  const int lane = threadIdx.x & 31;
  long long acc = 0;
  if (lane == 0) stk[0] = pack_box(0, 0, W, H);
  int top = 1;
  __syncwarp();
  while (top > 0) {
    const uint64_t bx = stk[top - 1];
    top--;
    __syncwarp();  // every lane has read the popped entry before it is overwritten
    const int X0 = (int)(bx & 0xffff), Y0 = (int)((bx >> 16) & 0xffff);
    const int X1 = (int)((bx >> 32) & 0xffff), Y1 = (int)(bx >> 48);
    const int Wb = X1 - X0, Hb = Y1 - Y0;
    if ((long long)Wb * Hb < T) {
      acc += pixelize<COUNT>(X0, Y0, X1, Y1, P, Q, sp, sq, counters);
      continue;
    }
    const Split g = make_split(Wb, Hb);
    unsigned hp, pp, hq, pq;
    classify(P, P.dx - X0, P.dy - Y0, Wb, Hb, g, hp, pp);
    classify(Q, Q.dx - X0, Q.dy - Y0, Wb, Hb, g, hq, pq);
    const int cc = lane & (g.kx - 1), rr = lane >> g.lkx;
    const unsigned valid = __ballot_sync(FULL, cc < g.ncols && rr < g.nrows);
    const unsigned in_p = ~hp & pp, out_p = ~hp & ~pp, in_q = ~hq & pq, out_q = ~hq & ~pq;
    // BOXCONTRIBUTE / BOXCONTINUE (Alg. 1 l.33-35, reading R7)
    const unsigned contrib = valid & in_p & in_q;
    const unsigned cont = valid & ~(out_p | out_q) & ~contrib;
    const int x0 = cc << g.lsx, y0 = rr << g.lsy;
    const int x1 = min(x0 + (1 << g.lsx), Wb), y1 = min(y0 + (1 << g.lsy), Hb);
    if ((contrib >> lane) & 1u) acc += (long long)(x1 - x0) * (y1 - y0);
    const int ncont = __popc(cont);
    if (COUNT && lane == 0) {
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_BOXES], (unsigned long long)__popc(valid));
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_BOXEDGES],
                (unsigned long long)(P.nv + P.V + Q.nv + Q.V));
      atomicAdd((unsigned long long*)&counters[SCCG_CNT_SPLITS], 1ull);
    }
    if (top + ncont > kStackCap) {
      status |= SCCG_STATUS_STACK;
      break;
    }
    if ((cont >> lane) & 1u) stk[top + __popc(cont & lanemask_lt())] = pack_box(X0 + x0, Y0 + y0, X0 + x1, Y0 + y1);
    top += ncont;
    __syncwarp();
  }
  return acc;
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
template <bool COUNT>
__global__ void __launch_bounds__(kWarps * 32, 3)
    large_kernel(DevSet Ps, DevSet Qs, const int2* __restrict__ pairs, const long long* __restrict__ list,
                 const unsigned* __restrict__ count, long long* __restrict__ inter, long long* __restrict__ uni,
                 sccg_sums* sums, int T, int mode, unsigned long long* queue, long long* counters) {
  extern __shared__ int4 s_dyn[];  // [kWarps][2][kECap] edge scratch, then [kWarps][kStackCap] stack
  __shared__ unsigned long long s_red[kWarps][11];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int4* sp = s_dyn + (size_t)warp * 2 * kECap;
  int4* sq = sp + kECap;
  uint64_t* stk = reinterpret_cast<uint64_t*>(s_dyn + (size_t)kWarps * 2 * kECap) + (size_t)warp * kStackCap;
  const long long n = *count;
  unsigned long long a_n = 0, a_nz = 0, a_i = 0, a_u = 0, a_ap = 0, a_aq = 0, limb[4] = {0, 0, 0, 0};
  unsigned status = 0;
  for (;;) {
    unsigned long long i0 = 0;
    if (lane == 0) i0 = atomicAdd(queue, 1ull);
    i0 = __shfl_sync(FULL, i0, 0);
    if ((long long)i0 >= n) break;
    const long long k = list[i0];
    const int2 pq = pairs[k];
    const int4 mp = Ps.mbr[pq.x], mq = Qs.mbr[pq.y];
    const int bx0 = max(mp.x, mq.x), by0 = max(mp.y, mq.y);
    const int bx1 = min(mp.z, mq.z), by1 = min(mp.w, mq.w);
    const int2 cp = Ps.ecount[pq.x], cq = Qs.ecount[pq.y];
    PairCtx P, Q;
    const long long op = Ps.off[pq.x], oq = Qs.off[pq.y];
    P.ev = Ps.edges + op;
    P.v = Ps.xy + op;
    P.V = (int)(Ps.off[pq.x + 1] - op);
    P.nv = cp.x;
    P.nh = cp.y;
    P.dx = mp.x - bx0;
    P.dy = mp.y - by0;
    P.ox = bx0;
    P.oy = by0;
    Q.ev = Qs.edges + oq;
    Q.v = Qs.xy + oq;
    Q.V = (int)(Qs.off[pq.y + 1] - oq);
    Q.nv = cq.x;
    Q.nh = cq.y;
    Q.dx = mq.x - bx0;
    Q.dy = mq.y - by0;
    Q.ox = bx0;
    Q.oy = by0;
    const int W = bx1 - bx0, H = by1 - by0;
    if (COUNT && lane == 0) atomicAdd((unsigned long long*)&counters[SCCG_CNT_ROOTPX], (unsigned long long)W * H);
    long long acc;
    if (mode == 1 || (long long)W * H < T)
      acc = pixelize<COUNT>(0, 0, W, H, P, Q, sp, sq, counters);
    else
      acc = sample<COUNT>(W, H, P, Q, stk, sp, sq, T, counters, status);
    const long long I = warp_sum64(acc);
    if (lane == 0) {
      const long long ap = Ps.area[pq.x], aq = Qs.area[pq.y];
      const long long U = ap + aq - I;  // indirect union
      if (inter) inter[k] = I;
      if (uni) uni[k] = U;
      a_n++;
      a_i += I;
      a_ap += ap;
      a_aq += aq;
      if (I != 0) {
        a_nz++;
        a_u += U;
        add_ratio_limbs(I, U, limb);
      }
    }
  }
  if (lane == 0) {
    s_red[warp][0] = a_n;
    s_red[warp][1] = a_nz;
    s_red[warp][2] = a_i;
    s_red[warp][3] = a_u;
    s_red[warp][4] = a_ap;
    s_red[warp][5] = a_aq;
    for (int i = 0; i < 4; i++) s_red[warp][6 + i] = limb[i];
    s_red[warp][10] = status;
  }
  __syncthreads();
  if (threadIdx.x < 11) {
    unsigned long long v = 0;
    for (int w = 0; w < kWarps; w++) v = threadIdx.x == 10 ? (v | s_red[w][10]) : v + s_red[w][threadIdx.x];
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(sums);
    if (threadIdx.x == 10) {
      if (v) atomicOr(&dst[10], v);
    } else if (v) {
      atomicAdd(&dst[threadIdx.x], v);
    }
  }
}

// --------------------------------------------------------------- small pairs
// The common case (nucleus pairs): root box at most 32 x 32 pixels and below
// T, each polygon at most kSmallCap vertical edges.  A warp claims 32 pairs,
// loads their metadata lane-parallel (32 independent loads in flight), then
// walks them with a software pipeline: while pair j is pixelized, pair j+1's
// edge records are already in flight into registers.  Pixelization is one row
// per lane (one 32-bit row word), half-warp per polygon when the box has at
// most 16 rows.  Per-pair results and sums are written lane-parallel.
constexpr int kSmallWarps = 8;
constexpr int kSmallCap = 64;   // vertical edges per polygon on this path
constexpr int kSmallQOff = 72;  // q buffer offset in records (8 B): 576 B, so p[t] and q[t] hit different banks

// Stage one polygon's row-crossing edges for a box of H <= 32 rows and
// W <= 32 columns as {row bits, pixel mask}: bit r of `rows` is set iff the
// edge crosses row r of the box (ylo <= r < yhi), `mask` holds the pixels the
// edge toggles.  Edges crossing no row are culled; every slot of the 32-record
// block (64 with `two`) is written -- kept records first, then zero records
// (no-ops) -- so no padding pass is needed.  Returns the loop length.
__device__ __forceinline__ int stage_rows(uint64_t r0, uint64_t r1, int nv, bool two, int dx, int dy, int H,
                                          int2* buf) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  int c, lo, hi;
  unpack_edge(r0, c, lo, hi);
  unsigned rows = low_bits(min(hi + dy, H)) & ~low_bits(lo + dy);
  bool keep = lane < nv && rows != 0;
  unsigned b = __ballot_sync(FULL, keep);
  int cnt = __popc(b);
  buf[keep ? __popc(b & lt) : cnt + __popc(~b & lt)] =
      keep ? make_int2((int)rows, (int)suffix_mask(c + dx)) : make_int2(0, 0);
  if (!two) return cnt;
  unpack_edge(r1, c, lo, hi);
  rows = low_bits(min(hi + dy, H)) & ~low_bits(lo + dy);
  keep = lane + 32 < nv && rows != 0;
  b = __ballot_sync(FULL, keep);
  cnt = __popc(b);
  buf[32 + (keep ? __popc(b & lt) : cnt + __popc(~b & lt))] =
      keep ? make_int2((int)rows, (int)suffix_mask(c + dx)) : make_int2(0, 0);
  return 32 + cnt;
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

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

#ifndef SCCG_SMALL_MINB
#define SCCG_SMALL_MINB 4
#endif
template <bool COUNT>
__global__ void __launch_bounds__(kSmallWarps * 32, SCCG_SMALL_MINB)
    small_kernel(DevSet Ps, DevSet Qs, const int2* __restrict__ pairs, long long n_cap,
                 const long long* __restrict__ dev_result, long long* __restrict__ inter,
                 long long* __restrict__ uni, sccg_sums* sums, int T, int mode, unsigned long long* queue,
                 long long* __restrict__ large_list, unsigned* large_count, long long* counters, long long np_,
                 long long nq_) {
  // pair count: host-given, or (async path) the filter's device-side count clamped to the buffer
  const long long n = dev_result ? min(dev_result[0], n_cap) : n_cap;
  if (dev_result && blockIdx.x == 0 && threadIdx.x == 0 && dev_result[1])
    atomicOr(reinterpret_cast<unsigned long long*>(&sums->status), (unsigned long long)dev_result[1]);
  __shared__ __align__(16) int2 s_buf[kSmallWarps][2 * kSmallQOff];
  __shared__ int4 s_meta[kSmallWarps][32];
  __shared__ int2 s_ep[kSmallWarps][32];
  __shared__ unsigned long long s_acc[kSmallWarps][16];
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
    if (k < n) {
      pq = pairs[k];
      ok = (unsigned)pq.x < (unsigned long long)np_ && (unsigned)pq.y < (unsigned long long)nq_;
      if (!ok) status |= SCCG_STATUS_ARG;  // index out of range: pair skipped
    }
    if (ok) {
      const int4 mp = Ps.mbr[pq.x], mq = Qs.mbr[pq.y];
      const int2 cp = Ps.ecount[pq.x], cq = Qs.ecount[pq.y];
      const long long op = Ps.off[pq.x], oq = Qs.off[pq.y];
      const int bx0 = max(mp.x, mq.x), by0 = max(mp.y, mq.y);
      const int W = min(mp.z, mq.z) - bx0, H = min(mp.w, mq.w) - by0;
      const int dxp = mp.x - bx0, dyp = mp.y - by0, dxq = mq.x - bx0, dyq = mq.y - by0;
      empty = !(W > 0 && H > 0);  // reading R18: I = 0
      small = !empty && W <= 32 && H <= 32 && (mode == 1 || W * H < T) && cp.x <= kSmallCap && cq.x <= kSmallCap &&
              op + cp.x < (1ll << 31) && oq + cq.x < (1ll << 31) && min(min(dxp, dyp), min(dxq, dyq)) >= -32768;
      meta[lane] = make_int4((int)((unsigned)W | ((unsigned)H << 6) | ((unsigned)cp.x << 12) | ((unsigned)cq.x << 20)),
                             (int)(((unsigned)dxp & 0xffffu) | ((unsigned)dyp << 16)),
                             (int)(((unsigned)dxq & 0xffffu) | ((unsigned)dyq << 16)), 0);
      epq[lane] = make_int2((int)op, (int)oq);
    }
    __syncwarp();
    // ---- everything else goes to the generic kernel (warp-aggregated append)
    const bool large = ok && !empty && !small;
    const unsigned lb = __ballot_sync(FULL, large);
    if (lb) {
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(large_count, (unsigned)__popc(lb));
      base = __shfl_sync(FULL, base, 0);
      if (large) large_list[base + __popc(lb & lanemask_lt())] = k;
    }
    // ---- small pairs, software-pipelined: records of the next pair are in
    // flight into registers while the current pair is pixelized
    unsigned todo = __ballot_sync(FULL, small);
    unsigned myI = 0;
    uint64_t np0 = 0, np1 = 0, nq0 = 0, nq1 = 0;
    auto prefetch = [&](int j) {
      const unsigned mj = (unsigned)meta[j].x;
      const int2 e = epq[j];
      const int nvp = (mj >> 12) & 127, nvq = (mj >> 20) & 127;
      const uint64_t* pe = Ps.edges + e.x;
      const uint64_t* qe = Qs.edges + e.y;
      np0 = lane < nvp ? __ldg(pe + lane) : 0ull;
      nq0 = lane < nvq ? __ldg(qe + lane) : 0ull;
      if (nvp > 32) np1 = lane + 32 < nvp ? __ldg(pe + 32 + lane) : 0ull;
      if (nvq > 32) nq1 = lane + 32 < nvq ? __ldg(qe + 32 + lane) : 0ull;
    };
    if (todo) prefetch(__ffs(todo) - 1);
    unsigned long long c_tests = 0, c_px = 0;
    const unsigned bit0 = 1u << (lane & 15), bit1 = 1u << ((lane & 15) + 16);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t cp0 = np0, cp1 = np1, cq0 = nq0, cq1 = nq1;
      if (todo) prefetch(__ffs(todo) - 1);
      const int4 mm = meta[j];
      const unsigned mj = (unsigned)mm.x, dpj = (unsigned)mm.y, dqj = (unsigned)mm.z;
      const int W = mj & 63, H = (mj >> 6) & 63, nvp = (mj >> 12) & 127, nvq = (mj >> 20) & 127;
      const bool two = max(nvp, nvq) > 32;
      const int cntp = stage_rows(cp0, cp1, nvp, two, (int)(short)(dpj & 0xffffu), (int)dpj >> 16, H, bp);
      const int cntq = stage_rows(cq0, cq1, nvq, two, (int)(short)(dqj & 0xffffu), (int)dqj >> 16, H, bq);
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
      const unsigned I = __reduce_add_sync(FULL, cnt);
      if (lane == j) myI = I;
      if (COUNT) {
        c_tests += (unsigned long long)H * (cntp + cntq);
        c_px += (unsigned long long)W * H;
      }
      __syncwarp();  // buffers are rewritten by the next pair
    }
    // ---- lane-parallel outputs and batch totals
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
        a[12] += c_px;
        a[13] += n_small;
      }
    }
  }
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
  unsigned long long* queue;  // [2] small, large
  unsigned* large_count;
  long long* large_list;
};

static size_t pixelbox_layout(int64_t n, Carve& cv, PixelboxWs& w) {
  w.queue = cv.take<unsigned long long>(4);
  w.large_count = reinterpret_cast<unsigned*>(w.queue + 2);
  w.large_list = cv.take<long long>(n > 0 ? n : 1);
  return cv.used;
}

size_t pixelbox_ws_bytes(int64_t n) {
  Carve cv{nullptr, ~size_t(0)};
  PixelboxWs w;
  return pixelbox_layout(n, cv, w) + 256;
}

constexpr size_t kDynSmem = (size_t)kWarps * (2 * kECap * sizeof(int4) + kStackCap * sizeof(uint64_t));

static cudaError_t prepare_kernels() {
  static cudaError_t once = [] {
    cudaError_t e = cudaFuncSetAttribute(large_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(large_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynSmem);
    return e;
  }();
  return once;
}

int run_pixelbox(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n,
                 const int64_t* dev_result, int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg,
                 void* ws, size_t ws_bytes, cudaStream_t stream) {
  Carve cv{reinterpret_cast<char*>(ws), ws_bytes};
  PixelboxWs w;
  pixelbox_layout(n, cv, w);
  if (!cv.ok || ws == nullptr) return set_error(SCCG_E_WORKSPACE, "pixelbox workspace too small");
  int T = cfg && cfg->threshold > 0 ? cfg->threshold : 2048;
  const int mode = cfg ? cfg->mode : 0;
  if (T < 2) T = 2;
  if (mode != 0 && mode != 1) return set_error(SCCG_E_ARG, "config.mode must be 0 (PixelBox) or 1 (PixelOnly)");
  cudaMemsetAsync(w.queue, 0, 4 * sizeof(unsigned long long), stream);
  if (n == 0) return check_cuda(cudaGetLastError(), "pixelbox");
  const bool count = cfg && cfg->counters;
  long long* counters = count ? reinterpret_cast<long long*>(cfg->counters) : nullptr;
  if (int r = check_cuda(prepare_kernels(), "pixelbox smem attribute")) return r;
  static int sms = 0, per_sm_s[2] = {0, 0}, per_sm_l[2] = {0, 0};
  if (sms == 0) {  // launch geometry, queried once
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s[1], small_kernel<true>, kSmallWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l[1], large_kernel<true>, kWarps * 32, kDynSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s[0], small_kernel<false>, kSmallWarps * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l[0], large_kernel<false>, kWarps * 32, kDynSmem);
  }
  int64_t grid_s = cfg && cfg->grid > 0 ? cfg->grid : (int64_t)sms * max(per_sm_s[count], 1);
  const int64_t need = (n + kSmallWarps * 32 - 1) / (kSmallWarps * 32);
  if (grid_s > need) grid_s = need;
  if (grid_s < 1) grid_s = 1;
  int64_t grid_l = cfg && cfg->grid > 0 ? cfg->grid : (int64_t)sms * max(per_sm_l[count], 1);
  const int64_t need_l = (n + kWarps - 1) / kWarps;
  if (grid_l > need_l) grid_l = need_l;
  if (grid_l < 1) grid_l = 1;
  DevSet Ps = dev_set(p), Qs = dev_set(q);
  const int2* pr = reinterpret_cast<const int2*>(pairs);
  long long* in = reinterpret_cast<long long*>(inter);
  long long* un = reinterpret_cast<long long*>(uni);
  const long long* dr = reinterpret_cast<const long long*>(dev_result);
  if (count) {
    small_kernel<true><<<(unsigned)grid_s, kSmallWarps * 32, 0, stream>>>(
        Ps, Qs, pr, n, dr, in, un, sums, T, mode, w.queue, w.large_list, w.large_count, counters, p->n_polygons,
        q->n_polygons);
    large_kernel<true><<<(unsigned)grid_l, kWarps * 32, kDynSmem, stream>>>(Ps, Qs, pr, w.large_list, w.large_count,
                                                                          in, un, sums, T, mode, w.queue + 1, counters);
  } else {
    small_kernel<false><<<(unsigned)grid_s, kSmallWarps * 32, 0, stream>>>(
        Ps, Qs, pr, n, dr, in, un, sums, T, mode, w.queue, w.large_list, w.large_count, nullptr, p->n_polygons,
        q->n_polygons);
    large_kernel<false><<<(unsigned)grid_l, kWarps * 32, kDynSmem, stream>>>(Ps, Qs, pr, w.large_list, w.large_count,
                                                                           in, un, sums, T, mode, w.queue + 1, nullptr);
  }
  return check_cuda(cudaGetLastError(), "pixelbox launch");
}

}  // namespace sccg
