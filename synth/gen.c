/* synth/gen.c -- seeded synthetic polygon sets for SCCG / PixelBox tests and bench.
 *
 * INPUT GENERATION ONLY.  This module holds none of the method's arithmetic: no
 * point-in-polygon test, no polygon area, no intersection, no MBR join and no
 * Jaccard.  It draws parametric blobs (nucleus / gland shapes) onto small pixel
 * masks, cleans each mask into a simply-connected 4-connected region without
 * diagonal pinches, and traces the region's outer boundary into a
 * counter-clockwise rectilinear ring (integer vertices, axis-parallel edges, one
 * vertex per change of direction).  It is the only code that both oracle/ and the
 * CUDA path consume (their inputs), per the task's independence rule.
 *
 * The workload recipe follows PAPER.md §5.1:
 * "The average size of polygons is about 150 in the number of pixels contained,
 * with the standard deviation around 100", whole-slide images pre-partitioned
 * into tiles (§2.1), and two result sets that are two segmentations of the
 * same image (§2.1).  Randomness is a counter-based splitmix64 stream keyed
 * by (seed, tile, stream id), so output is identical for any thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ RNG */
typedef struct { uint64_t s; } rng_t;

static inline uint64_t rng_next(rng_t* r) {
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static rng_t rng_make(uint64_t seed, uint64_t a, uint64_t b) {
  rng_t r;
  r.s = seed * 0xD1B54A32D192ED03ULL ^ (a + 1) * 0x9E3779B97F4A7C15ULL ^ (b + 7) * 0xC2B2AE3D27D4EB4FULL;
  rng_next(&r);
  rng_next(&r);
  return r;
}
static inline double u01(rng_t* r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline double uab(rng_t* r, double a, double b) { return a + (b - a) * u01(r); }
static inline int iab(rng_t* r, int a, int b) { /* inclusive */
  return a + (int)(rng_next(r) % (uint64_t)(b - a + 1));
}
static double nrm(rng_t* r) {
  double u = u01(r), v = u01(r);
  if (u < 1e-300) u = 1e-300;
  return sqrt(-2.0 * log(u)) * cos(2.0 * M_PI * v);
}

/* --------------------------------------------------------- output buffer */
typedef struct {
  int32_t* xy;  /* [nv][2] */
  int64_t nv, cap_v;
  int64_t* off; /* [np+1] */
  int64_t np, cap_p;
  int want_masks;
  int32_t* mbox; /* [np][4]: x0, y0, w, h of the exported mask */
  uint8_t* mbits;
  int64_t nm, cap_m;
  int64_t* moff; /* [np+1] */
} pbuf;

static void* xrealloc(void* p, size_t n) {
  void* q = realloc(p, n ? n : 1);
  if (!q) abort();
  return q;
}
static void pbuf_init(pbuf* b, int want_masks) {
  memset(b, 0, sizeof(*b));
  b->want_masks = want_masks;
  b->cap_p = 64;
  b->off = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (b->cap_p + 1));
  b->off[0] = 0;
  if (want_masks) {
    b->moff = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (b->cap_p + 1));
    b->moff[0] = 0;
    b->mbox = (int32_t*)xrealloc(NULL, sizeof(int32_t) * 4 * b->cap_p);
  }
}
static void pbuf_free(pbuf* b) {
  free(b->xy);
  free(b->off);
  free(b->mbox);
  free(b->mbits);
  free(b->moff);
  memset(b, 0, sizeof(*b));
}
static void pbuf_push_vertex(pbuf* b, int32_t x, int32_t y) {
  if (b->nv == b->cap_v) {
    b->cap_v = b->cap_v ? b->cap_v * 2 : 1024;
    b->xy = (int32_t*)xrealloc(b->xy, sizeof(int32_t) * 2 * b->cap_v);
  }
  b->xy[2 * b->nv] = x;
  b->xy[2 * b->nv + 1] = y;
  b->nv++;
}
static void pbuf_close_polygon(pbuf* b) {
  if (b->np + 1 >= b->cap_p) {
    b->cap_p *= 2;
    b->off = (int64_t*)xrealloc(b->off, sizeof(int64_t) * (b->cap_p + 1));
    if (b->want_masks) {
      b->moff = (int64_t*)xrealloc(b->moff, sizeof(int64_t) * (b->cap_p + 1));
      b->mbox = (int32_t*)xrealloc(b->mbox, sizeof(int32_t) * 4 * b->cap_p);
    }
  }
  b->np++;
  b->off[b->np] = b->nv;
}
/* append all of src after dst (tile concatenation in tile order) */
static void pbuf_append(pbuf* d, const pbuf* s) {
  for (int64_t i = 0; i < s->np; i++) {
    for (int64_t v = s->off[i]; v < s->off[i + 1]; v++) pbuf_push_vertex(d, s->xy[2 * v], s->xy[2 * v + 1]);
    if (d->want_masks) {
      int64_t len = s->moff[i + 1] - s->moff[i];
      if (d->nm + len > d->cap_m) {
        while (d->nm + len > d->cap_m) d->cap_m = d->cap_m ? d->cap_m * 2 : 4096;
        d->mbits = (uint8_t*)xrealloc(d->mbits, d->cap_m);
      }
      memcpy(d->mbits + d->nm, s->mbits + s->moff[i], (size_t)len);
      d->nm += len;
    }
    pbuf_close_polygon(d);
    if (d->want_masks) {
      memcpy(d->mbox + 4 * (d->np - 1), s->mbox + 4 * i, 4 * sizeof(int32_t));
      d->moff[d->np] = d->nm;
    }
  }
}

/* ------------------------------------------------------------------ grids */
/* cell (i, j) of a grid is the global pixel (ox + i, oy + j); m[j * w + i] */
typedef struct {
  int w, h, ox, oy;
  uint8_t* m;
} grid_t;

static void grid_alloc(grid_t* g, int w, int h, int ox, int oy) {
  g->w = w;
  g->h = h;
  g->ox = ox;
  g->oy = oy;
  g->m = (uint8_t*)calloc((size_t)w * h, 1);
  if (!g->m) abort();
}
static void grid_free(grid_t* g) {
  free(g->m);
  g->m = NULL;
}

/* keep only the largest 4-connected foreground component; returns its size */
static int64_t keep_largest(grid_t* g, int32_t* stack, int32_t* label) {
  const int w = g->w, h = g->h;
  int64_t n = (int64_t)w * h, best = 0;
  int32_t best_lab = -1, lab = 0;
  for (int64_t i = 0; i < n; i++) label[i] = -1;
  for (int64_t s = 0; s < n; s++) {
    if (!g->m[s] || label[s] >= 0) continue;
    int64_t sz = 0, sp = 0;
    stack[sp++] = (int32_t)s;
    label[s] = lab;
    while (sp) {
      int32_t c = stack[--sp];
      sz++;
      int x = c % w, y = c / w;
      int nb[4] = {c - 1, c + 1, c - w, c + w};
      int ok[4] = {x > 0, x < w - 1, y > 0, y < h - 1};
      for (int k = 0; k < 4; k++)
        if (ok[k] && g->m[nb[k]] && label[nb[k]] < 0) {
          label[nb[k]] = lab;
          stack[sp++] = nb[k];
        }
    }
    if (sz > best) {
      best = sz;
      best_lab = lab;
    }
    lab++;
  }
  for (int64_t i = 0; i < n; i++) g->m[i] = (label[i] == best_lab) ? 1 : 0;
  return best;
}

/* background cells not 4-connected to the grid border become foreground */
static int fill_holes(grid_t* g, int32_t* stack, int32_t* label) {
  const int w = g->w, h = g->h;
  int64_t n = (int64_t)w * h, sp = 0;
  int changed = 0;
  for (int64_t i = 0; i < n; i++) label[i] = 0;
  for (int x = 0; x < w; x++) {
    int64_t a = x, b = (int64_t)(h - 1) * w + x;
    if (!g->m[a] && !label[a]) { label[a] = 1; stack[sp++] = (int32_t)a; }
    if (!g->m[b] && !label[b]) { label[b] = 1; stack[sp++] = (int32_t)b; }
  }
  for (int y = 0; y < h; y++) {
    int64_t a = (int64_t)y * w, b = (int64_t)y * w + w - 1;
    if (!g->m[a] && !label[a]) { label[a] = 1; stack[sp++] = (int32_t)a; }
    if (!g->m[b] && !label[b]) { label[b] = 1; stack[sp++] = (int32_t)b; }
  }
  while (sp) {
    int32_t c = stack[--sp];
    int x = c % w, y = c / w;
    int nb[4] = {c - 1, c + 1, c - w, c + w};
    int ok[4] = {x > 0, x < w - 1, y > 0, y < h - 1};
    for (int k = 0; k < 4; k++)
      if (ok[k] && !g->m[nb[k]] && !label[nb[k]]) {
        label[nb[k]] = 1;
        stack[sp++] = nb[k];
      }
  }
  for (int64_t i = 0; i < n; i++)
    if (!g->m[i] && !label[i]) {
      g->m[i] = 1;
      changed = 1;
    }
  return changed;
}

/* a 2x2 window holding exactly a diagonal pair is a pinch; fill one off cell */
static int fix_pinches(grid_t* g) {
  const int w = g->w, h = g->h;
  int changed = 0;
  for (int y = 0; y + 1 < h; y++)
    for (int x = 0; x + 1 < w; x++) {
      uint8_t* a = &g->m[(int64_t)y * w + x];
      uint8_t* b = a + 1;
      uint8_t* c = a + w;
      uint8_t* d = c + 1;
      if (*a && *d && !*b && !*c) { *b = 1; changed = 1; }
      else if (*b && *c && !*a && !*d) { *a = 1; changed = 1; }
    }
  return changed;
}

/* Make the foreground one simply-connected, pinch-free 4-connected region whose
 * boundary is a single simple closed curve.  Foreground must not touch the
 * one-cell border of the grid.  Returns the cell count (0 = empty). */
static int64_t clean_region(grid_t* g) {
  int64_t n = (int64_t)g->w * g->h;
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* label = (int32_t*)malloc(sizeof(int32_t) * n);
  if (!stack || !label) abort();
  int64_t cnt = keep_largest(g, stack, label);
  if (cnt > 0) {
    for (int it = 0; it < 64; it++) {
      int c1 = fill_holes(g, stack, label);
      int c2 = fix_pinches(g);
      if (!c1 && !c2) break;
    }
    cnt = 0;
    for (int64_t i = 0; i < n; i++) cnt += g->m[i];
  }
  free(stack);
  free(label);
  return cnt;
}

/* Trace the boundary of a cleaned region counter-clockwise (interior on the
 * left, y up) and append it to b as one ring; one vertex per direction change.
 * Start: lower-left corner of the lowest, then leftmost, foreground cell. */
static void trace_ring(const grid_t* g, pbuf* b) {
  const int w = g->w, h = g->h, W = w + 1;
  /* out-direction per grid corner: 0:+x 1:+y 2:-x 3:-y, -1 none */
  int8_t* out = (int8_t*)malloc((size_t)(w + 1) * (h + 1));
  if (!out) abort();
  memset(out, -1, (size_t)(w + 1) * (h + 1));
  int sx = -1, sy = -1;
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) {
      if (!g->m[(int64_t)y * w + x]) continue;
      if (sx < 0) { sx = x; sy = y; }
      int below = (y > 0) && g->m[(int64_t)(y - 1) * w + x];
      int right = (x < w - 1) && g->m[(int64_t)y * w + x + 1];
      int above = (y < h - 1) && g->m[(int64_t)(y + 1) * w + x];
      int left = (x > 0) && g->m[(int64_t)y * w + x - 1];
      if (!below) out[(int64_t)y * W + x] = 0;
      if (!right) out[(int64_t)y * W + x + 1] = 1;
      if (!above) out[(int64_t)(y + 1) * W + x + 1] = 2;
      if (!left) out[(int64_t)(y + 1) * W + x] = 3;
    }
  static const int dx[4] = {1, 0, -1, 0}, dy[4] = {0, 1, 0, -1};
  int x = sx, y = sy, prev = 3; /* arriving from above along the left edge */
  do {
    int d = out[(int64_t)y * W + x];
    if (d != prev) pbuf_push_vertex(b, g->ox + x, g->oy + y);
    prev = d;
    x += dx[d];
    y += dy[d];
  } while (!(x == sx && y == sy));
  pbuf_close_polygon(b);
  free(out);
}

/* record the mask of the last closed polygon (pin data for tests) */
static void export_mask(const grid_t* g, pbuf* b) {
  if (!b->want_masks) return;
  int x0 = g->w, y0 = g->h, x1 = -1, y1 = -1;
  for (int y = 0; y < g->h; y++)
    for (int x = 0; x < g->w; x++)
      if (g->m[(int64_t)y * g->w + x]) {
        if (x < x0) x0 = x;
        if (x > x1) x1 = x;
        if (y < y0) y0 = y;
        if (y > y1) y1 = y;
      }
  int mw = x1 - x0 + 1, mh = y1 - y0 + 1;
  int64_t len = (int64_t)mw * mh;
  if (b->nm + len > b->cap_m) {
    while (b->nm + len > b->cap_m) b->cap_m = b->cap_m ? b->cap_m * 2 : 4096;
    b->mbits = (uint8_t*)xrealloc(b->mbits, b->cap_m);
  }
  for (int y = 0; y < mh; y++)
    for (int x = 0; x < mw; x++) b->mbits[b->nm + (int64_t)y * mw + x] = g->m[(int64_t)(y + y0) * g->w + x + x0];
  b->nm += len;
  int64_t i = b->np - 1;
  b->mbox[4 * i + 0] = g->ox + x0;
  b->mbox[4 * i + 1] = g->oy + y0;
  b->mbox[4 * i + 2] = mw;
  b->mbox[4 * i + 3] = mh;
  b->moff[b->np] = b->nm;
}

/* ------------------------------------------------------------------ blobs */
#define NHARM_MAX 16
typedef struct {
  double cx, cy; /* center (pixel-corner coordinates) */
  double ra, rb; /* semi-axes */
  double th;     /* major-axis angle */
  int nh;        /* harmonics k = 2 .. nh+1 */
  double c[NHARM_MAX], ps[NHARM_MAX];
} blob_t;

#define RTAB_MAX 4096
/* radius table over [0, 2pi); n entries scale with the blob's perimeter */
static void blob_rtab(const blob_t* bl, double* tab, int n) {
  for (int i = 0; i < n; i++) {
    double phi = 2.0 * M_PI * i / n, r = 1.0;
    for (int k = 0; k < bl->nh; k++) r += bl->c[k] * cos((k + 2) * phi + bl->ps[k]);
    tab[i] = r < 0.3 ? 0.3 : r;
  }
}
static double blob_rmax(const blob_t* bl) {
  double s = 1.0;
  for (int k = 0; k < bl->nh; k++) s += fabs(bl->c[k]);
  return (bl->ra > bl->rb ? bl->ra : bl->rb) * s + 2.0;
}
/* rasterize: cell center (x + 1/2, y + 1/2) inside the noisy ellipse.  The grid
 * gets a 2-cell empty border.  side = -1/0/+1 keeps u<0 / all / u>=0 (splits). */
static void blob_raster(const blob_t* bl, grid_t* g, int side) {
  double R = blob_rmax(bl), tab[RTAB_MAX];
  int ntab = (int)(8.0 * R);
  if (ntab < 64) ntab = 64;
  if (ntab > RTAB_MAX) ntab = RTAB_MAX;
  blob_rtab(bl, tab, ntab);
  double tmin = tab[0], tmax = tab[0];
  for (int i = 1; i < ntab; i++) {
    if (tab[i] < tmin) tmin = tab[i];
    if (tab[i] > tmax) tmax = tab[i];
  }
  int x0 = (int)floor(bl->cx - R) - 2, y0 = (int)floor(bl->cy - R) - 2;
  int x1 = (int)ceil(bl->cx + R) + 2, y1 = (int)ceil(bl->cy + R) + 2;
  grid_alloc(g, x1 - x0 + 1, y1 - y0 + 1, x0, y0);
  double ct = cos(bl->th), st = sin(bl->th);
  for (int j = 2; j < g->h - 2; j++)
    for (int i = 2; i < g->w - 2; i++) {
      double px = x0 + i + 0.5 - bl->cx, py = y0 + j + 0.5 - bl->cy;
      double u = px * ct + py * st, v = -px * st + py * ct;
      if (side < 0 && u >= 0) continue;
      if (side > 0 && u < 0) continue;
      double a = u / bl->ra, b = v / bl->rb;
      double rho = sqrt(a * a + b * b);
      if (rho <= tmin) { g->m[(int64_t)j * g->w + i] = 1; continue; }
      if (rho > tmax) continue;
      double phi = atan2(b, a);
      if (phi < 0) phi += 2.0 * M_PI;
      double t = phi * (ntab / (2.0 * M_PI));
      int k0 = (int)t;
      double f = t - k0;
      double rr = tab[k0 % ntab] * (1 - f) + tab[(k0 + 1) % ntab] * f;
      if (rho <= rr) g->m[(int64_t)j * g->w + i] = 1;
    }
}

/* lognormal area with mean 150, sd 100, clipped to [lo, hi] */
static double nucleus_area(rng_t* r, double mean, double sd, double lo, double hi) {
  double s2 = log(1.0 + (sd * sd) / (mean * mean));
  double mu = log(mean) - 0.5 * s2;
  double a = exp(mu + sqrt(s2) * nrm(r));
  if (a < lo) a = lo;
  if (a > hi) a = hi;
  return a;
}
static void fresh_harmonics(rng_t* r, blob_t* bl, int nh, double sd) {
  bl->nh = nh;
  for (int k = 0; k < nh; k++) {
    bl->c[k] = sd * nrm(r) / sqrt((double)nh) * (nh > 4 ? 2.0 / (k + 2) : 1.0);
    bl->ps[k] = uab(r, 0, 2 * M_PI);
  }
}
static void nucleus_params(rng_t* r, blob_t* bl, double cx, double cy) {
  double A = nucleus_area(r, 150.0, 100.0, 12.0, 1000.0);
  double asp = uab(r, 1.0, 1.8);
  bl->cx = cx;
  bl->cy = cy;
  bl->ra = sqrt(A * asp / M_PI);
  bl->rb = sqrt(A / (asp * M_PI));
  bl->th = uab(r, 0, M_PI);
  fresh_harmonics(r, bl, 4, 0.15);
}
static void gland_params(rng_t* r, blob_t* bl, double cx, double cy) {
  double side = uab(r, 64.0, 512.0), asp = uab(r, 1.0, 1.6);
  bl->cx = cx;
  bl->cy = cy;
  bl->ra = 0.5 * side / 1.25;
  bl->rb = bl->ra / asp;
  bl->th = uab(r, 0, M_PI);
  fresh_harmonics(r, bl, 11, 0.30); /* orders 2..12 */
}

/* morphological 4-neighbourhood dilation (d > 0) or erosion (d < 0), |d| steps */
static void morph(grid_t* g, int d) {
  int w = g->w, h = g->h;
  uint8_t* t = (uint8_t*)malloc((size_t)w * h);
  if (!t) abort();
  for (int s = 0; s < (d > 0 ? d : -d); s++) {
    memcpy(t, g->m, (size_t)w * h);
    for (int y = 1; y < h - 1; y++)
      for (int x = 1; x < w - 1; x++) {
        int64_t c = (int64_t)y * w + x;
        uint8_t n4o = t[c - 1] | t[c + 1] | t[c - w] | t[c + w];
        uint8_t n4a = t[c - 1] & t[c + 1] & t[c - w] & t[c + w];
        g->m[c] = d > 0 ? (t[c] | n4o) : (t[c] & n4a);
      }
  }
  free(t);
}
/* grow a grid by `pad` empty cells on every side */
static void grid_pad(grid_t* g, int pad) {
  grid_t n;
  grid_alloc(&n, g->w + 2 * pad, g->h + 2 * pad, g->ox - pad, g->oy - pad);
  for (int y = 0; y < g->h; y++) memcpy(n.m + (int64_t)(y + pad) * n.w + pad, g->m + (int64_t)y * g->w, g->w);
  grid_free(g);
  *g = n;
}

/* ------------------------------------------------------------ occupancy */
typedef struct {
  int x0, y0, w, h;
  uint64_t* bits;
} occ_t;
static void occ_init(occ_t* o, int x0, int y0, int w, int h) {
  o->x0 = x0;
  o->y0 = y0;
  o->w = w;
  o->h = h;
  o->bits = (uint64_t*)calloc(((size_t)w * h + 63) / 64, 8);
  if (!o->bits) abort();
}
static inline int occ_get(const occ_t* o, int x, int y) {
  int64_t i = (int64_t)(y - o->y0) * o->w + (x - o->x0);
  return (int)((o->bits[i >> 6] >> (i & 63)) & 1);
}
static inline void occ_set(occ_t* o, int x, int y) {
  int64_t i = (int64_t)(y - o->y0) * o->w + (x - o->x0);
  o->bits[i >> 6] |= 1ULL << (i & 63);
}
/* region fits in the occupancy window (1-px inset) and overlaps nothing */
static int occ_fits(const occ_t* o, const grid_t* g) {
  for (int j = 0; j < g->h; j++)
    for (int i = 0; i < g->w; i++) {
      if (!g->m[(int64_t)j * g->w + i]) continue;
      int x = g->ox + i, y = g->oy + j;
      if (x < o->x0 + 1 || y < o->y0 + 1 || x >= o->x0 + o->w - 1 || y >= o->y0 + o->h - 1) return 0;
      if (occ_get(o, x, y)) return 0;
    }
  return 1;
}
static void occ_commit(occ_t* o, const grid_t* g) {
  for (int j = 0; j < g->h; j++)
    for (int i = 0; i < g->w; i++)
      if (g->m[(int64_t)j * g->w + i]) occ_set(o, g->ox + i, g->oy + j);
}
/* Clip a region against cells already owned by other polygons of the same set
 * (touching neighbours in a segmentation share a border, never a pixel).
 * Cells outside the occupancy window are dropped too.  Returns kept cells. */
static int64_t occ_clip(const occ_t* o, grid_t* g) {
  int64_t kept = 0;
  for (int j = 0; j < g->h; j++)
    for (int i = 0; i < g->w; i++) {
      uint8_t* c = &g->m[(int64_t)j * g->w + i];
      if (!*c) continue;
      int x = g->ox + i, y = g->oy + j;
      if (x < o->x0 + 1 || y < o->y0 + 1 || x >= o->x0 + o->w - 1 || y >= o->y0 + o->h - 1 || occ_get(o, x, y))
        *c = 0;
      else
        kept++;
    }
  return kept;
}

/* try to emit a cleaned region into set b under occupancy o; consumes g.
 * The region is clipped against owned cells; it is rejected if less than
 * half of it survives or cleaning would re-enter an owned cell. */
static int emit_region(grid_t* g, occ_t* o, pbuf* b) {
  int ok = 0;
  int64_t before = 0;
  for (int64_t i = 0; i < (int64_t)g->w * g->h; i++) before += g->m[i];
  int64_t kept = occ_clip(o, g);
  if (2 * kept >= before && clean_region(g) > 0 && occ_fits(o, g)) {
    occ_commit(o, g);
    trace_ring(g, b);
    export_mask(g, b);
    ok = 1;
  }
  grid_free(g);
  return ok;
}

/* ------------------------------------------------------------------ spec */
typedef struct {
  uint64_t seed;
  int32_t x0, y0, width, height; /* image region */
  int32_t tile;                  /* tile side (P:67 tiles) */
  int32_t margin;                /* keep nuclei centers this far inside a tile */
  double nuclei_per_tile;        /* per full tile, set A */
  double cluster_frac;           /* fraction of nuclei placed in dense clusters */
  double spacing;                /* min center spacing of isolated nuclei */
  double cl_lo, cl_hi;           /* cluster member spacing range */
  int32_t glands_per_tile;       /* large glandular regions per tile (config 3) */
  double gland_split_frac;       /* glands that set B segments as nuclei */
  double drop_frac, split_frac, spur_frac; /* set-B perturbation mix */
  int32_t threads;
  int32_t want_masks;
} synth_spec;

typedef struct {
  int32_t* xy;
  int64_t* off;
  int64_t n_polygons, n_vertices;
  int32_t* mbox;
  uint8_t* mbits;
  int64_t* moff;
  int64_t n_maskbytes;
} synth_set;

typedef struct {
  synth_set a, b;
  int64_t rejected;
} synth_result;

typedef struct {
  const synth_spec* sp;
  int tx, ty;
  pbuf a, b;
  int64_t rejected;
} tile_job;

/* min-distance dart test against placed centers (linear scan over a cell hash) */
typedef struct {
  double* x;
  double* y;
  int n, cap;
} pts_t;
static void pts_push(pts_t* p, double x, double y) {
  if (p->n == p->cap) {
    p->cap = p->cap ? 2 * p->cap : 256;
    p->x = (double*)xrealloc(p->x, sizeof(double) * p->cap);
    p->y = (double*)xrealloc(p->y, sizeof(double) * p->cap);
  }
  p->x[p->n] = x;
  p->y[p->n] = y;
  p->n++;
}
static int pts_far(const pts_t* p, double x, double y, double d) {
  double d2 = d * d;
  for (int i = 0; i < p->n; i++) {
    double ex = p->x[i] - x, ey = p->y[i] - y;
    if (ex * ex + ey * ey < d2) return 0;
  }
  return 1;
}

static void gen_tile(tile_job* J) {
  const synth_spec* sp = J->sp;
  int tx0 = sp->x0 + J->tx * sp->tile, ty0 = sp->y0 + J->ty * sp->tile;
  int tw = sp->tile, th = sp->tile;
  if (tx0 + tw > sp->x0 + sp->width) tw = sp->x0 + sp->width - tx0;
  if (ty0 + th > sp->y0 + sp->height) th = sp->y0 + sp->height - ty0;
  uint64_t tid = (uint64_t)J->ty * 1000003ULL + (uint64_t)J->tx;
  rng_t ra = rng_make(sp->seed, tid, 0), rb = rng_make(sp->seed, tid, 1);
  occ_t oa, ob;
  occ_init(&oa, tx0, ty0, tw, th);
  occ_init(&ob, tx0, ty0, tw, th);
  pbuf_init(&J->a, sp->want_masks);
  pbuf_init(&J->b, sp->want_masks);
  double frac = (double)tw * th / ((double)sp->tile * sp->tile);
  int m = sp->margin;
  if (tw <= 2 * m + 4 || th <= 2 * m + 4) goto done;

  /* ---- glands (set A first so nuclei avoid them) */
  blob_t* gl = NULL;
  int ngl = 0;
  if (sp->glands_per_tile > 0) {
    gl = (blob_t*)calloc(sp->glands_per_tile, sizeof(blob_t));
    pts_t gp = {0};
    for (int k = 0, tries = 0; k < sp->glands_per_tile && tries < 200 * sp->glands_per_tile; tries++) {
      blob_t bl;
      double cx = uab(&ra, tx0 + 300, tx0 + tw - 300), cy = uab(&ra, ty0 + 300, ty0 + th - 300);
      gland_params(&ra, &bl, cx, cy);
      if (!pts_far(&gp, cx, cy, 0.5 * 2.5 * bl.ra + 200)) continue;
      grid_t g;
      blob_raster(&bl, &g, 0);
      if (emit_region(&g, &oa, &J->a)) {
        pts_push(&gp, cx, cy);
        gl[ngl++] = bl;
        k++;
      } else
        J->rejected++;
    }
    free(gp.x);
    free(gp.y);
  }

  /* ---- nucleus centers: isolated darts + dense clusters */
  int n_target = (int)floor(sp->nuclei_per_tile * frac + 0.5);
  int n_cl = (int)floor(n_target * sp->cluster_frac + 0.5), n_iso = n_target - n_cl;
  pts_t cen = {0};
  for (int k = 0, tries = 0; k < n_iso && tries < 40 * n_iso + 100; tries++) {
    double cx = uab(&ra, tx0 + m, tx0 + tw - m), cy = uab(&ra, ty0 + m, ty0 + th - m);
    if (!pts_far(&cen, cx, cy, sp->spacing)) continue;
    pts_push(&cen, cx, cy);
    k++;
  }
  int placed_cl = 0;
  while (placed_cl < n_cl) {
    int csz = iab(&ra, 4, 12);
    double sx = uab(&ra, tx0 + m, tx0 + tw - m), sy = uab(&ra, ty0 + m, ty0 + th - m);
    int base = cen.n;
    pts_push(&cen, sx, sy);
    placed_cl++;
    for (int k = 1; k < csz && placed_cl < n_cl; k++) {
      int par = base + iab(&ra, 0, cen.n - base - 1);
      double ang = uab(&ra, 0, 2 * M_PI), d = uab(&ra, sp->cl_lo, sp->cl_hi);
      double cx = cen.x[par] + d * cos(ang), cy = cen.y[par] + d * sin(ang);
      if (cx < tx0 + m || cy < ty0 + m || cx > tx0 + tw - m || cy > ty0 + th - m) continue;
      pts_push(&cen, cx, cy);
      placed_cl++;
    }
  }

  /* ---- set A nuclei */
  blob_t* na = (blob_t*)malloc(sizeof(blob_t) * (cen.n + 1));
  int nna = 0;
  for (int k = 0; k < cen.n; k++) {
    blob_t bl;
    nucleus_params(&ra, &bl, cen.x[k], cen.y[k]);
    grid_t g;
    blob_raster(&bl, &g, 0);
    if (emit_region(&g, &oa, &J->a))
      na[nna++] = bl;
    else
      J->rejected++;
  }

  /* ---- set B: glands (dilated / eroded / jittered, or re-segmented as nuclei) */
  for (int k = 0; k < ngl; k++) {
    blob_t bl = gl[k];
    if (u01(&rb) < sp->gland_split_frac) {
      /* second segmentation splits the gland into nuclei placed over it */
      double R = 0.9 * (bl.ra < bl.rb ? bl.ra : bl.rb);
      pts_t gp = {0};
      for (int t = 0; t < 400; t++) {
        double ang = uab(&rb, 0, 2 * M_PI), rr = R * sqrt(u01(&rb));
        double cx = bl.cx + rr * cos(ang), cy = bl.cy + rr * sin(ang);
        if (!pts_far(&gp, cx, cy, 16.0)) continue;
        pts_push(&gp, cx, cy);
        blob_t nb;
        nucleus_params(&rb, &nb, cx, cy);
        grid_t g;
        blob_raster(&nb, &g, 0);
        if (!emit_region(&g, &ob, &J->b)) J->rejected++;
      }
      free(gp.x);
      free(gp.y);
    } else {
      bl.cx += iab(&rb, -2, 2);
      bl.cy += iab(&rb, -2, 2);
      int d = iab(&rb, 1, 3) * (u01(&rb) < 0.5 ? -1 : 1);
      grid_t g;
      blob_raster(&bl, &g, 0);
      grid_pad(&g, 4);
      morph(&g, d);
      if (!emit_region(&g, &ob, &J->b)) J->rejected++;
    }
  }

  /* ---- set B nuclei: matched / dropped / split, then spurious extras */
  for (int k = 0; k < nna; k++) {
    blob_t bl = na[k];
    double u = u01(&rb);
    if (u < sp->drop_frac) continue;
    bl.cx += iab(&rb, -2, 2);
    bl.cy += iab(&rb, -2, 2);
    double s = sqrt(uab(&rb, 0.8, 1.2));
    bl.ra *= s;
    bl.rb *= s;
    fresh_harmonics(&rb, &bl, 4, 0.15);
    if (u < sp->drop_frac + sp->split_frac) {
      for (int side = -1; side <= 1; side += 2) {
        grid_t g;
        blob_raster(&bl, &g, side);
        if (!emit_region(&g, &ob, &J->b)) J->rejected++;
      }
    } else {
      grid_t g;
      blob_raster(&bl, &g, 0);
      if (!emit_region(&g, &ob, &J->b)) J->rejected++;
    }
  }
  int n_sp = (int)floor(nna * sp->spur_frac + 0.5);
  for (int k = 0; k < n_sp; k++) {
    blob_t bl;
    double cx = uab(&rb, tx0 + m, tx0 + tw - m), cy = uab(&rb, ty0 + m, ty0 + th - m);
    nucleus_params(&rb, &bl, cx, cy);
    grid_t g;
    blob_raster(&bl, &g, 0);
    if (!emit_region(&g, &ob, &J->b)) J->rejected++;
  }
  free(na);
  free(cen.x);
  free(cen.y);
  free(gl);
done:
  free(oa.bits);
  free(ob.bits);
}

typedef struct {
  tile_job* jobs;
  int n;
  int next;
  pthread_mutex_t mu;
} pool_t;
static void* worker(void* arg) {
  pool_t* P = (pool_t*)arg;
  for (;;) {
    pthread_mutex_lock(&P->mu);
    int i = P->next++;
    pthread_mutex_unlock(&P->mu);
    if (i >= P->n) break;
    gen_tile(&P->jobs[i]);
  }
  return NULL;
}

static void export_set(pbuf* b, synth_set* s) {
  s->xy = b->xy;
  s->off = b->off;
  s->n_polygons = b->np;
  s->n_vertices = b->nv;
  s->mbox = b->mbox;
  s->mbits = b->mbits;
  s->moff = b->moff;
  s->n_maskbytes = b->nm;
}

/* Generate both result sets for one image region.  Tiles are generated in
 * parallel and concatenated in row-major tile order.  Caller frees with
 * synth_free. Returns 0. */
int synth_generate(const synth_spec* sp, synth_result* out) {
  int ntx = (sp->width + sp->tile - 1) / sp->tile, nty = (sp->height + sp->tile - 1) / sp->tile;
  int n = ntx * nty;
  tile_job* jobs = (tile_job*)calloc(n, sizeof(tile_job));
  for (int t = 0; t < n; t++) {
    jobs[t].sp = sp;
    jobs[t].tx = t % ntx;
    jobs[t].ty = t / ntx;
  }
  pool_t P = {jobs, n, 0, PTHREAD_MUTEX_INITIALIZER};
  int nt = sp->threads > 0 ? sp->threads : 1;
  if (nt > n) nt = n;
  pthread_t th[256];
  if (nt > 256) nt = 256;
  for (int i = 0; i < nt; i++) pthread_create(&th[i], NULL, worker, &P);
  for (int i = 0; i < nt; i++) pthread_join(th[i], NULL);
  pbuf A, B;
  pbuf_init(&A, sp->want_masks);
  pbuf_init(&B, sp->want_masks);
  int64_t rej = 0;
  for (int t = 0; t < n; t++) {
    pbuf_append(&A, &jobs[t].a);
    pbuf_append(&B, &jobs[t].b);
    rej += jobs[t].rejected;
    pbuf_free(&jobs[t].a);
    pbuf_free(&jobs[t].b);
  }
  free(jobs);
  export_set(&A, &out->a);
  export_set(&B, &out->b);
  out->rejected = rej;
  return 0;
}

void synth_free(synth_result* r) {
  synth_set* s[2] = {&r->a, &r->b};
  for (int i = 0; i < 2; i++) {
    free(s[i]->xy);
    free(s[i]->off);
    free(s[i]->mbox);
    free(s[i]->mbits);
    free(s[i]->moff);
  }
  memset(r, 0, sizeof(*r));
}

/* Trace one caller-supplied mask (w x h bytes, row-major, cell (i,j) = pixel
 * (ox+i, oy+j)) into a ring after cleaning.  Used by tests to build rings for
 * exhaustively enumerated polyominoes.  Writes at most cap vertices into xy
 * and returns the vertex count, 0 if empty, -1 if cap is too small.  The
 * cleaned mask is written back into `mask`. */
int synth_trace_mask(const uint8_t* mask, int w, int h, int ox, int oy, uint8_t* cleaned, int32_t* xy, int cap) {
  grid_t g;
  grid_alloc(&g, w + 2, h + 2, ox - 1, oy - 1);
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++) g.m[(int64_t)(y + 1) * g.w + x + 1] = mask[(int64_t)y * w + x] ? 1 : 0;
  int64_t cnt = clean_region(&g);
  int nv = 0;
  if (cnt > 0) {
    pbuf b;
    pbuf_init(&b, 0);
    trace_ring(&g, &b);
    nv = (int)b.nv;
    if (nv > cap)
      nv = -1;
    else
      memcpy(xy, b.xy, sizeof(int32_t) * 2 * b.nv);
    pbuf_free(&b);
  }
  if (cleaned)
    for (int y = 0; y < h; y++)
      for (int x = 0; x < w; x++) cleaned[(int64_t)y * w + x] = g.m[(int64_t)(y + 1) * g.w + x + 1];
  grid_free(&g);
  return nv;
}
