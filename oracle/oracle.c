/* oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the PixelBox
 * hot path of SCCG (arXiv 1208.0277).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or helper with paper_1208_0277_b200/ (the CUDA path), and the
 * CUDA path never calls it.
 *
 * Every function is the plain definition from PAPER.md, written out:
 *   - pixel model: pixel (x, y) is the unit cell [x, x+1) x [y, y+1); its
 *     position relative to a polygon is decided by casting a ray from the cell
 *     center and counting boundary crossings, odd = inside.  PAPER.md §3.1
 *     P:151-155 ("the coordinates of vertices are integer-valued ... cast a ray
 *     from the pixel and count its number of intersections with the polygon's
 *     boundary ... if the number is odd, the pixel lies inside").  The crossing
 *     test is the textbook even-odd (PNPOLY) test for an arbitrary polygon; it is
 *     NOT specialised to rectilinear edges.  DESIGN.md reading R1.
 *   - polygon area: the shoelace formula A = 1/2 sum(x_i y_{i+1} - x_{i+1} y_i),
 *     PAPER.md §3.2 P:193.
 *   - area of intersection / union of a pair: count the pixels of the pair's
 *     bounding region that lie inside both / inside either polygon, PAPER.md
 *     §3.1 P:153 (the three pixel categories).  Both are counted directly; the
 *     identity |p u q| = |p| + |q| - |p n q| is a test, not an input.
 *   - MBR join: every (p, q) whose half-open MBRs overlap (the `&&` predicate of
 *     Fig. 1(b); half-open reading R4), by nested loop and by a
 *     textbook x-sorted plane sweep; output sorted by (p, q).  The closed-box
 *     variant (touching MBRs pair too) feeds ST_Touches.
 *   - ST_Touches (reading R21): the closed polygons meet but their
 *     interiors do not.  Written out on the pixel model: no pixel lies in both
 *     (|p n q| = 0) and some pixel of p shares at least a corner with some
 *     pixel of q (their closed unit squares intersect) -- counted pixel by pixel,
 *     no edge arithmetic.
 * Parallelism: pairs are split statically across threads; results do not
 * depend on the split.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ PIP */
/* Even-odd crossing count of the ray from (px, py) toward +x (PNPOLY). */
int oracle_pip(const int32_t* xy, int64_t nv, double px, double py) {
  int c = 0;
  for (int64_t i = 0, j = nv - 1; i < nv; j = i++) {
    double xi = xy[2 * i], yi = xy[2 * i + 1], xj = xy[2 * j], yj = xy[2 * j + 1];
    if (((yi > py) != (yj > py)) && (px < (xj - xi) * (py - yi) / (yj - yi) + xi)) c = !c;
  }
  return c;
}

/* Pixel (x, y) inside polygon: ray from its center (x + 1/2, y + 1/2). */
int oracle_pixel_in(const int32_t* xy, int64_t nv, int32_t x, int32_t y) {
  return oracle_pip(xy, nv, (double)x + 0.5, (double)y + 0.5);
}

/* ---------------------------------------------------------------- area */
/* Shoelace: 1/2 |sum_i (x_i y_{i+1} - x_{i+1} y_i)|, int64. */
int64_t oracle_area_shoelace(const int32_t* xy, int64_t nv) {
  int64_t s = 0;
  for (int64_t i = 0; i < nv; i++) {
    int64_t j = (i + 1) % nv;
    s += (int64_t)xy[2 * i] * xy[2 * j + 1] - (int64_t)xy[2 * j] * xy[2 * i + 1];
  }
  if (s < 0) s = -s;
  return s / 2;
}

/* Vertex bounding box: [xmin, xmax) x [ymin, ymax) contains every pixel that
 * can lie inside (pixel centers lie strictly between vertex coordinates). */
void oracle_mbr(const int32_t* xy, int64_t nv, int32_t* out4) {
  int32_t x0 = xy[0], y0 = xy[1], x1 = xy[0], y1 = xy[1];
  for (int64_t i = 1; i < nv; i++) {
    if (xy[2 * i] < x0) x0 = xy[2 * i];
    if (xy[2 * i] > x1) x1 = xy[2 * i];
    if (xy[2 * i + 1] < y0) y0 = xy[2 * i + 1];
    if (xy[2 * i + 1] > y1) y1 = xy[2 * i + 1];
  }
  out4[0] = x0;
  out4[1] = y0;
  out4[2] = x1;
  out4[3] = y1;
}

/* ------------------------------------------------ row edge prefilter (exact) */
/* For one pixel row y, keep only the edges whose y-extent straddles the ray
 * ordinate y + 1/2 -- the only edges PNPOLY's first condition can accept -- and
 * run the same crossing test against them.  Equivalent to oracle_pip by
 * construction; tests check the two agree.  Scratch `ex` holds 4 doubles per
 * kept edge (xi, yi, xj, yj). */
static int64_t row_edges(const int32_t* xy, int64_t nv, double py, double* ex) {
  int64_t k = 0;
  for (int64_t i = 0, j = nv - 1; i < nv; j = i++) {
    double yi = xy[2 * i + 1], yj = xy[2 * j + 1];
    if ((yi > py) != (yj > py)) {
      ex[4 * k] = xy[2 * i];
      ex[4 * k + 1] = yi;
      ex[4 * k + 2] = xy[2 * j];
      ex[4 * k + 3] = yj;
      k++;
    }
  }
  return k;
}
static inline int row_pip(const double* ex, int64_t k, double px, double py) {
  int c = 0;
  for (int64_t e = 0; e < k; e++) {
    double xi = ex[4 * e], yi = ex[4 * e + 1], xj = ex[4 * e + 2], yj = ex[4 * e + 3];
    if (px < (xj - xi) * (py - yi) / (yj - yi) + xi) c = !c;
  }
  return c;
}

/* Pixel mask of a polygon over the window [x0, x0+w) x [y0, y0+h):
 * out[j*w+i] = pixel (x0+i, y0+j) inside.  mode 0 = plain PNPOLY per pixel,
 * mode 1 = row prefilter.  Returns the number of inside pixels. */
int64_t oracle_mask(const int32_t* xy, int64_t nv, int32_t x0, int32_t y0, int32_t w, int32_t h, uint8_t* out,
                    int mode) {
  int64_t cnt = 0;
  double* ex = mode ? (double*)malloc(sizeof(double) * 4 * (nv + 1)) : NULL;
  for (int32_t j = 0; j < h; j++) {
    double py = (double)(y0 + j) + 0.5;
    int64_t k = mode ? row_edges(xy, nv, py, ex) : 0;
    for (int32_t i = 0; i < w; i++) {
      double px = (double)(x0 + i) + 0.5;
      int in = mode ? row_pip(ex, k, px, py) : oracle_pip(xy, nv, px, py);
      if (out) out[(int64_t)j * w + i] = (uint8_t)in;
      cnt += in;
    }
  }
  free(ex);
  return cnt;
}

/* |p| by counting pixels of its vertex bounding box. */
int64_t oracle_area_pixels(const int32_t* xy, int64_t nv, int mode) {
  int32_t b[4];
  oracle_mbr(xy, nv, b);
  return oracle_mask(xy, nv, b[0], b[1], b[2] - b[0], b[3] - b[1], NULL, mode);
}

/* |p n q| and |p u q| by scanning every pixel of the bounding box of
 * MBR(p) u MBR(q): inside both -> intersection; inside either -> union. */
void oracle_pair(const int32_t* xp, int64_t np, const int32_t* xq, int64_t nq, int64_t* inter, int64_t* uni,
                 int mode) {
  int32_t a[4], b[4];
  oracle_mbr(xp, np, a);
  oracle_mbr(xq, nq, b);
  int32_t x0 = a[0] < b[0] ? a[0] : b[0], y0 = a[1] < b[1] ? a[1] : b[1];
  int32_t x1 = a[2] > b[2] ? a[2] : b[2], y1 = a[3] > b[3] ? a[3] : b[3];
  int64_t I = 0, U = 0;
  double* ep = mode ? (double*)malloc(sizeof(double) * 4 * (np + 1)) : NULL;
  double* eq = mode ? (double*)malloc(sizeof(double) * 4 * (nq + 1)) : NULL;
  for (int32_t y = y0; y < y1; y++) {
    double py = (double)y + 0.5;
    int64_t kp = mode ? row_edges(xp, np, py, ep) : 0, kq = mode ? row_edges(xq, nq, py, eq) : 0;
    for (int32_t x = x0; x < x1; x++) {
      double px = (double)x + 0.5;
      int ip = mode ? row_pip(ep, kp, px, py) : oracle_pip(xp, np, px, py);
      int iq = mode ? row_pip(eq, kq, px, py) : oracle_pip(xq, nq, px, py);
      I += ip & iq;
      U += ip | iq;
    }
  }
  free(ep);
  free(eq);
  *inter = I;
  *uni = U;
}

/* ------------------------------------------------------------ batches */
typedef struct {
  const int32_t *xyp, *xyq;
  const int64_t *offp, *offq;
  const int32_t* pairs;
  int64_t lo, hi;
  int64_t *inter, *uni;
  int mode;
} pair_job;

static void* pair_worker(void* arg) {
  pair_job* J = (pair_job*)arg;
  for (int64_t k = J->lo; k < J->hi; k++) {
    int64_t p = J->pairs[2 * k], q = J->pairs[2 * k + 1];
    oracle_pair(J->xyp + 2 * J->offp[p], J->offp[p + 1] - J->offp[p], J->xyq + 2 * J->offq[q],
                J->offq[q + 1] - J->offq[q], &J->inter[k], &J->uni[k], J->mode);
  }
  return NULL;
}

/* Areas of intersection / union for a batch of pairs (pairs[k] = (p, q)),
 * split statically over `threads` threads. */
void oracle_pairs(const int32_t* xyp, const int64_t* offp, const int32_t* xyq, const int64_t* offq,
                  const int32_t* pairs, int64_t n, int64_t* inter, int64_t* uni, int threads, int mode) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  pair_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t] = (pair_job){xyp, xyq, offp, offq, pairs, n * t / threads, n * (t + 1) / threads, inter, uni, mode};
    pthread_create(&th[t], NULL, pair_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
}

/* Per-polygon shoelace areas and vertex bounding boxes for a whole set. */
void oracle_set_props(const int32_t* xy, const int64_t* off, int64_t n, int64_t* area, int32_t* mbr) {
  for (int64_t i = 0; i < n; i++) {
    if (area) area[i] = oracle_area_shoelace(xy + 2 * off[i], off[i + 1] - off[i]);
    if (mbr) oracle_mbr(xy + 2 * off[i], off[i + 1] - off[i], mbr + 4 * i);
  }
}

/* --------------------------------------------------------------- join */
static inline int mbr_overlap(const int32_t* a, const int32_t* b) {
  /* half-open [x0, x1) x [y0, y1): overlap iff they share a pixel (reading R4) */
  return a[0] < b[2] && b[0] < a[2] && a[1] < b[3] && b[1] < a[3];
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* Nested loop over all (p, q).  Writes up to cap pairs (p-major, q-minor,
 * i.e. sorted) and returns the total count. */
int64_t oracle_join_nested(const int32_t* mbrp, int64_t np, const int32_t* mbrq, int64_t nq, int32_t* out,
                           int64_t cap) {
  int64_t n = 0;
  for (int64_t p = 0; p < np; p++)
    for (int64_t q = 0; q < nq; q++)
      if (mbr_overlap(mbrp + 4 * p, mbrq + 4 * q)) {
        if (n < cap) {
          out[2 * n] = (int32_t)p;
          out[2 * n + 1] = (int32_t)q;
        }
        n++;
      }
  return n;
}

typedef struct {
  int32_t x0;
  int32_t set; /* 0 = P, 1 = Q */
  int64_t id;
} ev_t;
static int cmp_ev(const void* a, const void* b) {
  const ev_t *x = (const ev_t*)a, *y = (const ev_t*)b;
  if (x->x0 != y->x0) return (x->x0 > y->x0) - (x->x0 < y->x0);
  if (x->set != y->set) return x->set - y->set;
  return (x->id > y->id) - (x->id < y->id);
}

/* Plane sweep in x: rectangles arrive in order of their left edge; each arrival
 * is tested against the still-open rectangles of the other set (those whose
 * right edge lies beyond the arrival's left edge), so every overlapping pair is
 * reported exactly once, by its later arrival.  Output sorted by (p, q).
 * Writes up to cap pairs, returns the total count. */
int64_t oracle_join_sweep(const int32_t* mbrp, int64_t np, const int32_t* mbrq, int64_t nq, int32_t* out,
                          int64_t cap) {
  int64_t ne = np + nq;
  ev_t* ev = (ev_t*)malloc(sizeof(ev_t) * (ne + 1));
  for (int64_t i = 0; i < np; i++) ev[i] = (ev_t){mbrp[4 * i], 0, i};
  for (int64_t i = 0; i < nq; i++) ev[np + i] = (ev_t){mbrq[4 * i], 1, i};
  qsort(ev, (size_t)ne, sizeof(ev_t), cmp_ev);
  int64_t *act[2], nact[2] = {0, 0};
  act[0] = (int64_t*)malloc(sizeof(int64_t) * (np + 1));
  act[1] = (int64_t*)malloc(sizeof(int64_t) * (nq + 1));
  const int32_t* M[2] = {mbrp, mbrq};
  int64_t n = 0, keycap = 1024;
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * keycap);
  for (int64_t e = 0; e < ne; e++) {
    int s = ev[e].set, o = 1 - s;
    const int32_t* r = M[s] + 4 * ev[e].id;
    /* drop closed rectangles of the other set */
    for (int64_t k = 0; k < nact[o];) {
      if (M[o][4 * act[o][k] + 2] <= r[0])
        act[o][k] = act[o][--nact[o]];
      else
        k++;
    }
    for (int64_t k = 0; k < nact[o]; k++) {
      const int32_t* t = M[o] + 4 * act[o][k];
      if (mbr_overlap(r, t)) {
        int64_t p = s == 0 ? ev[e].id : act[o][k], q = s == 0 ? act[o][k] : ev[e].id;
        if (n == keycap) {
          keycap *= 2;
          keys = (int64_t*)realloc(keys, sizeof(int64_t) * keycap);
        }
        keys[n++] = (p << 32) | q;
      }
    }
    act[s][nact[s]++] = ev[e].id;
  }
  qsort(keys, (size_t)n, sizeof(int64_t), cmp_i64);
  for (int64_t k = 0; k < n && k < cap; k++) {
    out[2 * k] = (int32_t)(keys[k] >> 32);
    out[2 * k + 1] = (int32_t)(keys[k] & 0xffffffff);
  }
  free(keys);
  free(act[0]);
  free(act[1]);
  free(ev);
  return n;
}

/* Nested loop over all (p, q) with CLOSED MBRs intersecting (touching boxes
 * included; the candidates of ST_Touches).  Sorted output, total returned. */
int64_t oracle_join_nested_closed(const int32_t* mbrp, int64_t np, const int32_t* mbrq, int64_t nq, int32_t* out,
                                  int64_t cap) {
  int64_t n = 0;
  for (int64_t p = 0; p < np; p++)
    for (int64_t q = 0; q < nq; q++) {
      const int32_t *a = mbrp + 4 * p, *b = mbrq + 4 * q;
      if (a[0] <= b[2] && b[0] <= a[2] && a[1] <= b[3] && b[1] <= a[3]) {
        if (n < cap) {
          out[2 * n] = (int32_t)p;
          out[2 * n + 1] = (int32_t)q;
        }
        n++;
      }
    }
  return n;
}

/* ST_Touches on the pixel model (reading R21): 1 iff no pixel is inside both
 * polygons and some pixel inside p and some pixel inside q are equal-or-
 * 8-adjacent (their closed unit squares meet).  Scans the bounding box of both
 * MBRs grown by one pixel; pixel classification by the PNPOLY ray test. */
int oracle_touches(const int32_t* xp, int64_t np, const int32_t* xq, int64_t nq) {
  int32_t a[4], b[4];
  oracle_mbr(xp, np, a);
  oracle_mbr(xq, nq, b);
  const int32_t x0 = (a[0] < b[0] ? a[0] : b[0]) - 1, y0 = (a[1] < b[1] ? a[1] : b[1]) - 1;
  const int32_t x1 = (a[2] > b[2] ? a[2] : b[2]) + 1, y1 = (a[3] > b[3] ? a[3] : b[3]) + 1;
  const int32_t w = x1 - x0, h = y1 - y0;
  uint8_t* mp = (uint8_t*)calloc((size_t)w * h, 1);
  uint8_t* mq = (uint8_t*)calloc((size_t)w * h, 1);
  oracle_mask(xp, np, x0, y0, w, h, mp, 0);
  oracle_mask(xq, nq, x0, y0, w, h, mq, 0);
  int both = 0, near = 0;
  for (int32_t j = 0; j < h; j++)
    for (int32_t i = 0; i < w; i++) {
      if (!mp[(int64_t)j * w + i]) continue;
      if (mq[(int64_t)j * w + i]) both = 1;
      for (int dj = -1; dj <= 1; dj++)
        for (int di = -1; di <= 1; di++) {
          const int32_t jj = j + dj, ii = i + di;
          if (jj >= 0 && jj < h && ii >= 0 && ii < w && mq[(int64_t)jj * w + ii]) near = 1;
        }
    }
  free(mp);
  free(mq);
  return !both && near;
}
