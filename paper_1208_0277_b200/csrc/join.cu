// join.cu -- MBR-overlap join by a hashed uniform grid, in
// four launches.
//
// The paper's filter stage searches a Hilbert R-tree on one CPU thread
// (§4.1) to produce "an array of polygon pairs with intersecting
// MBRs"; the predicate is the `&&` MBR test of Fig. 1(b), here
// half-open (reading R4).  On the GPU a uniform grid of 2^k-pixel cells is
// cheaper: Q's MBRs are inserted into every cell they cover, each P MBR probes
// its cells, and a pair is emitted only from the cell holding its reference
// point (max xlo, max ylo) so it is found exactly once.
//
//   1. grid_select_kernel -- clears the bucket counters and the overflow-pool
//      counter; one warp picks the cell size 2^k and the bucket wrap from the
//      per-set statistics sccg_prep gathered (no host round trip).
//   2. grid_insert_kernel -- each Q MBR takes a slot in the bucket of every
//      cell it covers (fixed-capacity buckets, an overflow chain past
//      kSlots): no count pass and no scan.
//   3. probe_kernel<false> -- thread per P (a warp per P that covers many
//      cells) counts its pairs, the CTA scans the counts and writes each P's
//      pairs, sorted by q, into the tile's own bucket.
//   4. probe_kernel<true> -- each tile sums the preceding tiles' counts for
//      its offset and copies its bucket into place: the output is sorted by
//      (p, q) without a global sort.  (A single pass with a decoupled
//      look-back was measured 2-3x slower: a tile whose P sit in a crowded
//      cluster holds back every tile after it, and the waiting CTAs hold the
//      SMs.)
//
// Cells are hashed onto 2^ax x 2^ay buckets by wrapping (a torus: bucket =
// (cy mod 2^ay, cx mod 2^ax)), so the cell size is not bound by the memory a
// dense grid over the whole slide would take; the wrap is at least as wide
// and tall as the largest Q MBR's cell span, so no Q MBR lands twice in one
// bucket, which -- with the reference-point rule -- keeps every pair emitted
// exactly once (proof in DESIGN.md §6, "join").
#include "internal.cuh"

namespace sccg {

struct __align__(16) Grid {
  int k, ax, ay, empty;
  __device__ __forceinline__ int bucket(int cx, int cy) const {
    return ((cy & ((1 << ay) - 1)) << ax) | (cx & ((1 << ax) - 1));
  }
};

// The grid is written by the selection kernel two launches earlier: read it
// with an L1-bypassing load (ld.global.cg), never through the read-only /
// L1 path -- under programmatic dependent launch a CTA that started early
// could otherwise see a stale copy of a recycled workspace (measured: a
// previous join's grid at the same address).
__device__ __forceinline__ Grid load_grid(const Grid* gp) {
  const int4 v = __ldcg(reinterpret_cast<const int4*>(gp));
  return Grid{v.x, v.y, v.z, v.w};
}

__device__ __forceinline__ bool mbr_empty(const int4& m) { return m.x >= m.z || m.y >= m.w; }

// A bucket's entries live in kLevels levels of kLevelSlots slots: entry j of
// bucket b is slot (j / kLevelSlots, b, j % kLevelSlots) of a level-major
// array, so the first four entries of neighbouring buckets share cache lines
// (level 0 is the dense part; the higher levels are touched only by crowded
// buckets), and every slot address is known before the bucket's count is
// read.  Past kSlots entries an overflow chain takes the rest.
#ifndef SCCG_JOIN_CSTRIDE
#define SCCG_JOIN_CSTRIDE 1  // bucket counters per int of spacing (8: one per 32-byte sector)
#endif
constexpr int kCStride = SCCG_JOIN_CSTRIDE;
#ifndef SCCG_JOIN_LEVELS
#define SCCG_JOIN_LEVELS 8
#endif
#ifndef SCCG_JOIN_LS
#define SCCG_JOIN_LS 4  // slots per level (4 or 8)
#endif
constexpr int kLevelSlots = SCCG_JOIN_LS, kLevels = SCCG_JOIN_LEVELS * 4 / SCCG_JOIN_LS,
              kSlots = kLevelSlots * kLevels;
static_assert(kLevelSlots == 4 || kLevelSlots == 8, "4 or 8 slots per level");
// 2^hb buckets, hb = ceil(log2(max(nq, 512))) (+ SCCG_JOIN_HB_EXTRA)
#ifndef SCCG_JOIN_HB_EXTRA
#define SCCG_JOIN_HB_EXTRA 0
#endif
static int bucket_bits(int64_t nq) {
  int b = 9;
  while (b < 27 && (int64_t(1) << b) < nq) b++;
  return b + SCCG_JOIN_HB_EXTRA;
}
// An entry: a Q MBR (grown for the closed join) and its index in 16 bytes --
// {xlo, ylo, (w - 1) | (h - 1) << 16, q} (w, h <= 65536 after growing).
__device__ __forceinline__ int4 pack_entry(const int4& m, int q) {
  return make_int4(m.x, m.y, (int)((unsigned)(m.z - m.x - 1) | ((unsigned)(m.w - m.y - 1) << 16)), q);
}
__device__ __forceinline__ int4 entry_box(const int4& e) {
  return make_int4(e.x, e.y, e.x + (int)((unsigned)e.z & 0xffffu) + 1, e.y + (int)((unsigned)e.z >> 16) + 1);
}
// overflow pool: the grid selection only accepts cell sizes whose upper bound
// on Q's cell incidences fits it, so it never runs out
static int64_t entry_cap(int64_t nq) { return 8 * nq + 1024; }

// Upper bound and expectation of the 2^k-cell incidences of one set
// (SetStats).  `grow` = 1: the boxes are grown by one pixel on the high side
// (closed join).
__device__ __forceinline__ void set_entries(const SetStats* s, int k, int grow, double& bound, double& expect) {
  const double c = 1.0 / (double)(1ll << k), n = (double)s->nonempty;
  const double sw = (double)s->sw + grow * n, sh = (double)s->sh + grow * n;
  const double swh = (double)s->swh + grow * ((double)s->sw + (double)s->sh + n);
  const double cont = swh * c * c + 2.0 * (sw + sh) * c + 4.0 * n;
  const double ext = n * (double)(((s->maxext[0] - 1 + grow) >> k) + 2) * (double)(((s->maxext[1] - 1 + grow) >> k) + 2);
  bound = cont < ext ? cont : ext;
  expect = n + (sw + sh) * c + swh * c * c;
}

__device__ __forceinline__ int ceil_log2(long long v) {
  int b = 0;
  while ((1ll << b) < v) b++;
  return b;
}

// Cell size 2^k and bucket wrap.  Lane j evaluates k = 3 + j: the expected
// work E_p + E_q + E_p * L / W (cell visits and inserts, candidate tests),
// where the candidates per visit L = E_q / min(cells, buckets).  Cell visits
// and inserts are dependent round trips (an atomic each for an insert) while
// a candidate test is one more load in flight: W = 10 is fitted to the
// measured join times of C2 and C3 at k = 5..9 ("join").
// (SCCG_JOIN_PACK=1 adds a packing estimate of clustered nuclei -- the
// number of Q MBRs of mean size w x h meeting a cell of side s when they tile
// the plane, (s + w)(s + h) / (w h) / 4; measured slower: it picks smaller
// cells, and more incidences cost more than the extra candidates.)
// Feasible: the wrap covers the largest Q MBR's cell span and the incidence
// bound fits the overflow pool; k = 30 always is.
#ifndef SCCG_JOIN_PACK
#define SCCG_JOIN_PACK 0
#endif
#ifndef SCCG_JOIN_TESTW
#define SCCG_JOIN_TESTW 10.0
#endif
__global__ void grid_select_kernel(const SetStats* __restrict__ sp, const SetStats* __restrict__ sq, int hb,
                                   long long ecap, int grow, Grid* g, int4* __restrict__ zero, long long zero_n4) {
  // No global access before the wait: under programmatic dependent launch
  // this kernel starts while its predecessor drains, and the workspace may be
  // memory a caching allocator just recycled from a buffer that predecessor
  // still reads (clearing before the wait zeroed live data; measured).
  pdl_entry();  // prep's statistics (and, for what follows, everything before)
  // every CTA clears its share of the bucket counters ...
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < zero_n4; i += (long long)gridDim.x * blockDim.x)
    zero[i] = make_int4(0, 0, 0, 0);
  const int lane = threadIdx.x & 31;
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const bool empty = sp->nonempty == 0 || sq->nonempty == 0;
  const int xmin = min(sp->bounds[0], sq->bounds[0]), ymin = min(sp->bounds[1], sq->bounds[1]);
  const int xmax = max(sp->bounds[2], sq->bounds[2]) + grow, ymax = max(sp->bounds[3], sq->bounds[3]) + grow;
  const int k = 3 + lane;
  double cost = 1e300;
  int ax = 0;
  if (!empty && k <= 30) {
    const long long ncx = (long long)(((xmax - 1) >> k) - (xmin >> k) + 1);
    const long long ncy = (long long)(((ymax - 1) >> k) - (ymin >> k) + 1);
    const int need_x = ceil_log2(((sq->maxext[0] - 1 + grow) >> k) + 2);
    const int need_y = ceil_log2(((sq->maxext[1] - 1 + grow) >> k) + 2);
    ax = min(max(ceil_log2(ncx), need_x), hb - need_y);
    double bp, ep, bq, eq;
    set_entries(sp, k, grow, bp, ep);
    set_entries(sq, k, grow, bq, eq);
#ifdef SCCG_JOIN_FORCE_K
    if (k != SCCG_JOIN_FORCE_K) ax = -1;
#endif
    if (ax >= need_x && bq <= (double)ecap) {
      const double C = (double)ncx * (double)ncy, H = (double)(1ll << hb);
      const double s = (double)(1ll << k), n = (double)sq->nonempty;
      const double w = (double)sq->sw / n + 1.0 + grow, h = (double)sq->sh / n + 1.0 + grow;
      const double uni = eq / (C < H ? C : H), pack = 0.25 * (s + w) * (s + h) / (w * h);
      cost = ep + eq + ep * (SCCG_JOIN_PACK ? (uni > pack ? uni : pack) : uni) / SCCG_JOIN_TESTW;
    }
  }
  // argmin (ties -> smaller k); k = 30 is always feasible
  int best = k <= 30 ? k : 30, bax = ax;
  double bc = cost;
  for (int o = 16; o; o >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, bc, o);
    const int ok = __shfl_xor_sync(0xffffffffu, best, o);
    const int oa = __shfl_xor_sync(0xffffffffu, bax, o);
    if (oc < bc || (oc == bc && ok < best)) {
      bc = oc;
      best = ok;
      bax = oa;
    }
  }
  if (lane == 0) {
    Grid r{30, 1, hb - 1, 0};
    if (empty) {
      r.empty = 1;
    } else if (bc < 1e300) {
      r.k = best;
      r.ax = bax;
      r.ay = hb - bax;
    }
    *g = r;
  }
}

// MBRs covering more than kCoopCells cells (a gland among nuclei, C3) are
// inserted and probed by their whole warp, lanes spread over the cells, so
// one polygon is not a serial critical path of hundreds of cell visits.
#ifndef SCCG_COOP_CELLS
#define SCCG_COOP_CELLS 4
#endif
constexpr int kCoopCells = SCCG_COOP_CELLS;

__device__ __forceinline__ int mbr_cells(const int4& m, int k) {
  return (((m.z - 1) >> k) - (m.x >> k) + 1) * (((m.w - 1) >> k) - (m.y >> k) + 1);
}

// The hashed grid: bucket b holds count[b] entries, the first kSlots in its
// slots (level-major, see kLevelSlots), the rest in a chain through the
// overflow pool starting at head[b] (most recent first; the probe follows
// exactly count[b] - kSlots links, so head needs no clearing).
struct Tables {
  int* count;
  int4* slot;  // [kLevels][H][kLevelSlots] packed entries
  int* head;
  int4* ovf;  // [E] packed entries
  int* ovf_next;
  int* ovf_n;
  int hb;
  __device__ __forceinline__ size_t at(int b, int j) const {
    constexpr int ls = kLevelSlots == 8 ? 3 : 2;
    return ((size_t)(j / kLevelSlots) << (hb + ls)) + ((size_t)b << ls) + (j % kLevelSlots);
  }
};

// Insert Q: each MBR (grown for the closed join) takes a slot in the bucket of
// every cell it covers.
__global__ void grid_insert_kernel(const int4* __restrict__ mq, int64_t nq, const Grid* __restrict__ gp, Tables t,
                                   int grow) {
  pdl_entry();
  const Grid g = load_grid(gp);
  if (g.empty) return;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  auto place = [&](int b, int j, const int4& e) {  // entry j of bucket b
    if (j < kSlots) {
      t.slot[t.at(b, j)] = e;  // the probe tests MBRs straight from the bucket
    } else {
      const int o = atomicAdd(t.ovf_n, 1);
      t.ovf[o] = e;
      t.ovf_next[o] = atomicExch(&t.head[b], o);
    }
  };
  auto insert = [&](int cx, int cy, int q, const int4& m) {
    const int b = g.bucket(cx, cy);
    place(b, atomicAdd(&t.count[(size_t)b * kCStride], 1), pack_entry(m, q));
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
    if (ok && !coop) {  // at most kCoopCells cells: all slot claims in flight before the stores
      const int x0 = m.x >> g.k, y0 = m.y >> g.k, nx = ((m.z - 1) >> g.k) - x0 + 1;
      const int nc = nx * (((m.w - 1) >> g.k) - y0 + 1);
      int bk[kCoopCells], sl[kCoopCells];
#pragma unroll
      for (int c = 0; c < kCoopCells; c++) {
        bk[c] = g.bucket(x0 + c % nx, y0 + c / nx);
        sl[c] = c < nc ? atomicAdd(&t.count[(size_t)bk[c] * kCStride], 1) : 0;
      }
      const int4 e = pack_entry(m, (int)i);
#pragma unroll
      for (int c = 0; c < kCoopCells; c++)
        if (c < nc) place(bk[c], sl[c], e);
    }
    for (unsigned bm = __ballot_sync(0xffffffffu, coop); bm; bm &= bm - 1) {
      const int j = __ffs(bm) - 1;
      const int4 mj = make_int4(__shfl_sync(0xffffffffu, m.x, j), __shfl_sync(0xffffffffu, m.y, j),
                                __shfl_sync(0xffffffffu, m.z, j), __shfl_sync(0xffffffffu, m.w, j));
      const int qj = (int)(base + j);
      const int x0 = mj.x >> g.k, y0 = mj.y >> g.k, w = ((mj.z - 1) >> g.k) - x0 + 1;
      const int nc = w * (((mj.w - 1) >> g.k) - y0 + 1);
      for (int c = lane; c < nc; c += 32) insert(x0 + c % w, y0 + c / w, qj, mj);
    }
  }
}

#ifndef SCCG_PROBE_TILE
#define SCCG_PROBE_TILE 128
#endif
constexpr int kProbeTile = SCCG_PROBE_TILE;  // p per probe CTA
constexpr int kKeep = 4;                     // hits kept in registers by the counting pass

// (p, q) is owned by cell (cx, cy) iff the boxes overlap (half-open, R4) and
// the reference point (max xlo, max ylo) lies in that cell.
// With the cell bounds hoisted out of the entry loop: for a cell
// (cx, cy) that p covers, max(a.x, b.x) lies in column cx iff b.x < the
// column's end and -- unless cx is p's first column, where a.x already starts
// it -- b.x >= its start (a.x < the end of every column p covers); likewise y.
struct Own {
  int lx, hx, ly, hy;
};
__device__ __forceinline__ Own own_bounds(const int4& a, int k, int cx, int cy) {
  const long long ex = ((long long)cx + 1) << k, ey = ((long long)cy + 1) << k;
  return Own{cx == (a.x >> k) ? INT_MIN : (int)((long long)cx << k), (int)min(ex, (long long)INT_MAX),
             cy == (a.y >> k) ? INT_MIN : (int)((long long)cy << k), (int)min(ey, (long long)INT_MAX)};
}
__device__ __forceinline__ bool owns(const int4& a, const int4& b, const Own& o) {
  return a.x < b.z && b.x < a.z && a.y < b.w && b.y < a.w && b.x >= o.lx && b.x < o.hx && b.y >= o.ly && b.y < o.hy;
}

// Test one visited cell's bucket against `a`; take(h, q) for each entry
// tested (h: the entry is owned -- branch-free bookkeeping in the caller).
// The bucket's first two entries (one 32-byte sector) are loaded together
// with its count; loading a sector no insert wrote costs a DRAM miss, so the
// next ones only when the count says they exist.
#ifndef SCCG_JOIN_SPEC
#define SCCG_JOIN_SPEC 2
#endif
template <class Take>
__device__ __forceinline__ void visit(const int4& a, int k, int cx, int cy, int b, const Tables& t, Take&& take) {
  const int4* s0 = t.slot + t.at(b, 0);
  const int cnt = t.count[(size_t)b * kCStride];
  const Own o = own_bounds(a, k, cx, cy);
  const int4 e0 = s0[0];
#if SCCG_JOIN_SPEC >= 2
  const int4 e1 = s0[1];
#endif
  take(cnt > 0 && owns(a, entry_box(e0), o), e0.w);
  if (cnt > 1) {
#if SCCG_JOIN_SPEC < 2
    const int4 e1 = s0[1];
#endif
    take(owns(a, entry_box(e1), o), e1.w);
    if (cnt > 2) {
      const int4 e2 = s0[2], e3 = s0[3];
      take(owns(a, entry_box(e2), o), e2.w);
      take(cnt > 3 && owns(a, entry_box(e3), o), e3.w);
      if (kLevelSlots == 8 && cnt > 4) {  // the rest of the first level (one 128-byte line per bucket)
        const int4 e4 = s0[4], e5 = s0[5], e6 = s0[6], e7 = s0[7];
        take(owns(a, entry_box(e4), o), e4.w);
        take(cnt > 5 && owns(a, entry_box(e5), o), e5.w);
        take(cnt > 6 && owns(a, entry_box(e6), o), e6.w);
        take(cnt > 7 && owns(a, entry_box(e7), o), e7.w);
      }
      if (cnt > kLevelSlots) {  // a crowded bucket: the higher levels, then the overflow chain
        const int ns = min(cnt, kSlots);
        for (int j = kLevelSlots; j < ns; j += 4) {  // four entries at a time (a level of 8 in two halves)
          const int4* s = t.slot + t.at(b, j);
          const int4 f0 = s[0], f1 = s[1], f2 = s[2], f3 = s[3];
          take(owns(a, entry_box(f0), o), f0.w);
          take(j + 1 < ns && owns(a, entry_box(f1), o), f1.w);
          take(j + 2 < ns && owns(a, entry_box(f2), o), f2.w);
          take(j + 3 < ns && owns(a, entry_box(f3), o), f3.w);
        }
        if (cnt > kSlots) {  // rare
          int oi = t.head[b];
          for (int r = kSlots; r < cnt; r++) {
            const int4 e = t.ovf[oi];
            take(owns(a, entry_box(e), o), e.w);
            oi = t.ovf_next[oi];
          }
        }
      }
    }
  }
}

// Visit p's cells (at most kCoopCells), one after the other.
template <class Take>
__device__ __forceinline__ void probe_cells(const int4& a, const Grid& g, const Tables& t, Take&& take) {
  const int k = g.k;
  for (int cy = a.y >> k; cy <= (a.w - 1) >> k; cy++)
    for (int cx = a.x >> k; cx <= (a.z - 1) >> k; cx++) visit(a, k, cx, cy, g.bucket(cx, cy), t, take);
}

// The (big MBR, cell) visits of a probe tile, flattened over its threads:
// visit v (v < nv) is cell v - cstart[j] of thread j's MBR, j the last thread
// with cstart[j] <= v (cstart non-decreasing in j; threads without a big MBR
// have empty ranges).  take(j, owned, q) for every entry tested.
template <class Take>
__device__ __forceinline__ void coop_visits(int nv, const int* cstart, const int4* __restrict__ mp, int64_t p0,
                                            const Grid& g, const Tables& t, int grow, Take&& take) {
  const int k = g.k;
  for (int v = threadIdx.x; v < nv; v += kProbeTile) {
    int j = 0;
    for (int s = kProbeTile / 2; s; s >>= 1)
      if (cstart[j + s] <= v) j += s;
    int4 a = mp[p0 + j];
    a.z += grow;
    a.w += grow;
    const int x0 = a.x >> k, y0 = a.y >> k, w = ((a.z - 1) >> k) - x0 + 1;
    const int c = v - cstart[j];
    const int cx = x0 + c % w, cy = y0 + c / w;
    visit(a, k, cx, cy, g.bucket(cx, cy), t, [&](bool h, int q) { take(j, h, q); });
  }
}

// Sort seg[0..n) by q (distinct within a segment) with the warp: a bitonic
// network in its ascending-only form (each merge starts by comparing i with
// its mirror i ^ (k - 1)), so positions >= n behave as +inf and are never
// touched -- no padding needed.  Up to kSortBuf keys are sorted in the warp's
// shared buffer; longer segments in place in global memory (L1/L2-resident).
constexpr int kSortBuf = 512;  // keys per warp buffer
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

__device__ void warp_sort_segment(int2* seg, int n, int* buf) {
  const int lane = threadIdx.x & 31;
  if (n <= 1) return;
  const int p = seg[0].x;
  if (n <= kSortBuf) {  // in the warp's own shared buffer
    for (int i = lane; i < n; i += 32) buf[i] = seg[i].y;
    __syncwarp();
    warp_bitonic<int>(n, [&](int i) { return buf[i]; }, [&](int i, int v) { buf[i] = v; });
    for (int i = lane; i < n; i += 32) seg[i] = make_int2(p, buf[i]);
  } else {
    __syncwarp();
    warp_bitonic<int>(n, [&](int i) { return seg[i].y; }, [&](int i, int v) { seg[i] = make_int2(p, v); });
  }
  __syncwarp();
}

__device__ __forceinline__ void insertion_sort_q(int2* seg, int n) {
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


#ifndef SCCG_PROBE_MINB
#define SCCG_PROBE_MINB 8
#endif
constexpr int kBucket = 1024;  // pairs per probe tile held in its bucket between the two passes

// Probe, per CTA tile of kProbeTile consecutive p (thread per p; MBRs over
// many cells by the tile's warps together).  Each thread counts the pairs its
// p owns -- keeping up to kKeep q in registers -- and the CTA scans the counts.
// BUCKET pass (COMPACT = false): the tile's pairs go to its own bucket of
// kBucket slots, each p's segment sorted by q, and its count to tile_cnt (no
// cross-CTA dependency).  COMPACT pass: each tile sums the preceding tiles'
// counts (all known by then; a few vectorized L2 loads per thread) for its
// offset and copies its bucket there -- or, when the tile overflowed its
// bucket, probes again and writes in place; the last tile writes the total
// (and the async result word).  Pairs past `cap` are not written (a p whose
// segment would cross it is skipped whole); the total is exact.
template <bool COMPACT>
__global__ void __launch_bounds__(kProbeTile, SCCG_PROBE_MINB)
    probe_kernel(const int4* __restrict__ mp, int64_t np, const Grid* __restrict__ gp, Tables t,
                 int* __restrict__ tile_cnt, int2* __restrict__ bucket, int2* __restrict__ pairs, long long cap,
                 long long* __restrict__ total, long long* __restrict__ result, const uint32_t* __restrict__ status_p,
                 const uint32_t* __restrict__ status_q, int grow) {
  __shared__ int s_warp[kProbeTile / 32];
  __shared__ long long s_sum[kProbeTile / 32];
  __shared__ int s_fillc[kProbeTile];   // big MBRs' segment fill counters
  __shared__ int s_cstart[kProbeTile];   // first (big MBR, cell) visit of each thread's MBR
  __shared__ int s_coopval[kProbeTile];  // big MBRs' pair count, then their segment start
  __shared__ int s_cw[kProbeTile / 32];
  __shared__ int s_sort[kProbeTile / 32][kSortBuf];
  __shared__ int s_long[kProbeTile];  // threads whose segment is longer than kThreadSortMax
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  pdl_entry();
  int2* dst;       // this tile's output: its bucket, or its final place
  long long room;  // slots available from dst
  if (COMPACT) {
    // this tile's offset: the preceding tiles' counts (all known by now; a
    // few vectorized L2 loads per thread)
    long long sum = 0;
    const int4* c4 = reinterpret_cast<const int4*>(tile_cnt);
#pragma unroll 4
    for (int i = threadIdx.x; i < (tile >> 2); i += kProbeTile) {  // unrolled: the loads go out together
      const int4 v = __ldcg(c4 + i);
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
    if (cnt == 0 || pairs == nullptr || off >= cap) return;
    if (cnt <= kBucket) {  // copy the bucket (already sorted)
      const int2* src = bucket + (size_t)tile * kBucket;
      const long long m = min((long long)cnt, cap - off);
      for (int i = threadIdx.x; i < m; i += kProbeTile) pairs[off + i] = src[i];
      return;
    }
    dst = pairs + off;  // overflowed tile: probe again, write in place
    room = cap - off;
  } else {
    dst = bucket + (size_t)tile * kBucket;
    room = kBucket;
  }
  const int64_t p = (int64_t)tile * kProbeTile + threadIdx.x;
  const Grid g = load_grid(gp);
  int4 a = make_int4(0, 0, 0, 0);
  const bool live = p < np && !g.empty;
  if (live) a = mp[p];
  const bool act = live && !mbr_empty(a);
  a.z += grow;  // closed join: boxes grown by one pixel on the high side
  a.w += grow;
  const bool coop = act && mbr_cells(a, g.k) > kCoopCells;  // big MBR: the warps probe it together
  int n = 0;
  int4 keep = make_int4(0, 0, 0, 0);
  if (act && !coop)
    probe_cells(a, g, t, [&](bool h, int q) {
      if (h) {  // rare (about one candidate in ten is owned): a branch, not selects per candidate
        keep.x = n == 0 ? q : keep.x;
        keep.y = n == 1 ? q : keep.y;
        keep.z = n == 2 ? q : keep.z;
        keep.w = n == 3 ? q : keep.w;
        n++;
      }
    });
  // Big MBRs of the whole tile (glands among nuclei, C3: often consecutive in
  // p): their (MBR, cell) visits are flattened over all the tile's threads --
  // thread v takes visit v, v + kProbeTile, ... -- so a tile holding many
  // glands is neither a serial walk per warp nor per gland.  s_cstart = the
  // exclusive scan of the big MBRs' cell counts in thread order; visit v
  // belongs to the last thread j with s_cstart[j] <= v.
  const int mycells = coop ? mbr_cells(a, g.k) : 0;
  int ncv = 0;  // visits in the tile
  if (__syncthreads_or(coop)) {
    int xc = mycells;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, xc, o);
      if (lane >= o) xc += y;
    }
    if (lane == 31) s_cw[warp] = xc;
    __syncthreads();
    int wb = 0;
    for (int w = 0; w < kProbeTile / 32; w++) {
      wb += w < warp ? s_cw[w] : 0;
      ncv += s_cw[w];
    }
    s_cstart[threadIdx.x] = wb + xc - mycells;
    if (coop) s_coopval[threadIdx.x] = 0;
    __syncthreads();
    coop_visits(ncv, s_cstart, mp, (int64_t)tile * kProbeTile, g, t, grow, [&](int j, bool h, int q) {
      (void)q;
      if (h) atomicAdd(&s_coopval[j], 1);
    });
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
    if (agg > kBucket) return;  // rare: the compaction pass probes this tile again
  }
  int2* seg = dst + base;
  const bool fits = n > 0 && base + n <= room;
  // big MBRs: gathered by all threads' visits (as above), unsorted
  if (ncv > 0) {
    if (coop) {
      s_coopval[threadIdx.x] = fits ? base : -1;
      s_fillc[threadIdx.x] = 0;
    }
    __syncthreads();
    coop_visits(ncv, s_cstart, mp, (int64_t)tile * kProbeTile, g, t, grow, [&](int j, bool h, int q) {
      if (h && s_coopval[j] >= 0) dst[s_coopval[j] + atomicAdd(&s_fillc[j], 1)] = make_int2((int)(tile * kProbeTile + j), q);
    });
    __syncthreads();  // the visits' writes are visible to the segment's own thread
    if (coop && fits && n <= kThreadSortMax) insertion_sort_q(seg, n);
  }
  if (fits && !coop) {
    if (n <= kKeep) {  // the counting pass kept them: sort in registers, write
      const int big = 0x7fffffff;  // pad the unused slots so a 4-sorting network applies
      int k0 = keep.x, k1 = n > 1 ? keep.y : big, k2 = n > 2 ? keep.z : big, k3 = n > 3 ? keep.w : big;
#define SCCG_CSWAP(U, V)      \
  {                           \
    const int lo = min(U, V); \
    V = max(U, V);            \
    U = lo;                   \
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
      int w = 0;
      probe_cells(a, g, t, [&](bool h, int q) {
        if (h) seg[w++] = make_int2((int)p, q);
      });
      if (n <= kThreadSortMax) insertion_sort_q(seg, n);
    }
  }
  // long segments (big MBRs, or many hits): dealt round-robin to the warps
  // (s_coopval / s_fillc reused: each one's start and length)
  const bool lng = fits && n > kThreadSortMax;
  int nlong = 0;
  if (__syncthreads_or(lng)) {
    const unsigned lm = __ballot_sync(0xffffffffu, lng);
    if (lane == 0) s_cw[warp] = __popc(lm);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < kProbeTile / 32; w++) {
      off += w < warp ? s_cw[w] : 0;
      nlong += s_cw[w];
    }
    if (lng) {
      s_long[off + __popc(lm & lanemask_lt())] = threadIdx.x;
      s_coopval[threadIdx.x] = base;
      s_fillc[threadIdx.x] = n;
    }
    __syncthreads();
    for (int c = warp; c < nlong; c += kProbeTile / 32) {
      const int j = s_long[c];
      warp_sort_segment(dst + s_coopval[j], s_fillc[j], s_sort[warp]);
    }
  }
}

// --------------------------------------------------------------------- host
static int64_t probe_tiles(int64_t np) { return (np + kProbeTile - 1) / kProbeTile; }

struct FilterWs {
  Grid* grid;
  Tables t;
  int* tile_cnt;  // [T] pairs per probe tile
  int2* bucket;   // [T][kBucket] per-tile pair buckets
  long long* total;
  char* zero;     // cleared by the grid selection: bucket counters, overflow pool counter
  size_t zero_bytes;
  int hb;
};

static size_t filter_layout(int64_t np, int64_t nq, Carve& cv, FilterWs& w) {
  const int hb = bucket_bits(nq);
  const int64_t H = int64_t(1) << hb, E = entry_cap(nq), T = probe_tiles(np);
  w.hb = hb;
  w.grid = cv.take<Grid>(1);
  w.total = cv.take<long long>(1);
  // one contiguous cleared region: count[H] | pool counter
  const size_t cb = (size_t)4 * H * kCStride;
  w.zero_bytes = cb + 16;
  w.zero = cv.take<char>(w.zero_bytes);
  if (w.zero) {
    w.t.count = reinterpret_cast<int*>(w.zero);
    w.t.ovf_n = reinterpret_cast<int*>(w.zero + cb);
  }
  w.tile_cnt = cv.take<int>(T + 4);
  w.bucket = cv.take<int2>(T * kBucket);
  w.t.hb = hb;
  w.t.head = cv.take<int>(H);
  w.t.slot = cv.take<int4>(H * kSlots);
  w.t.ovf = cv.take<int4>(E);
  w.t.ovf_next = cv.take<int>(E);
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

__global__ void filter_result_kernel(long long* __restrict__ total, const uint32_t* __restrict__ sp,
                                     const uint32_t* __restrict__ sq, long long* result) {
  pdl_entry();
  if (threadIdx.x == 0) {
    *total = 0;
    if (result) {
      result[0] = 0;
      result[1] = (long long)(sp[0] | sq[0]);
    }
  }
}

// Enqueue the whole join: grid selection + clearing, Q insertion, one-pass
// probe (pairs written when their p's segment fits in `cap`; the exact total
// always lands in w.total).
static int filter_enqueue(const sccg_polyset* P, const sccg_polyset* Q, FilterWs& w, int32_t* pairs, int64_t cap,
                          long long* result, int grow, cudaStream_t stream) {
  const int64_t np = P->n_polygons, nq = Q->n_polygons;
  const int4* mp = reinterpret_cast<const int4*>(P->mbr);
  const int4* mq = reinterpret_cast<const int4*>(Q->mbr);
  const int64_t T = probe_tiles(np);
  const long long zero_n4 = (long long)(w.zero_bytes / 16);
  launch_pdl(grid_select_kernel, dim3((unsigned)blocks_for(zero_n4, 256)), dim3(256), 0, stream,
             reinterpret_cast<const SetStats*>(P->stats), reinterpret_cast<const SetStats*>(Q->stats), w.hb,
             (long long)entry_cap(nq), grow, w.grid, reinterpret_cast<int4*>(w.zero), zero_n4);
  if (nq > 0)
    launch_pdl(grid_insert_kernel, dim3(blocks_for(nq, 256)), dim3(256), 0, stream, mq, nq, w.grid, w.t, grow);
  if (np > 0) {
    launch_pdl(probe_kernel<false>, dim3((unsigned)T), dim3(kProbeTile), 0, stream, mp, np, w.grid, w.t, w.tile_cnt,
               w.bucket, (int2*)nullptr, (long long)0, (long long*)nullptr, (long long*)nullptr,
               (const uint32_t*)nullptr, (const uint32_t*)nullptr, grow);
    launch_pdl(probe_kernel<true>, dim3((unsigned)T), dim3(kProbeTile), 0, stream, mp, np, w.grid, w.t, w.tile_cnt,
               w.bucket, reinterpret_cast<int2*>(pairs), (long long)(pairs ? cap : 0), w.total, result, P->status,
               Q->status, grow);
  } else
    launch_pdl(filter_result_kernel, dim3(1), dim3(32), 0, stream, w.total, P->status, Q->status, result);
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
