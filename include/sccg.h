/* sccg.h -- C ABI of the B200-native PixelBox hot path of SCCG (arXiv 1208.0277).
 *
 * Operation (PAPER.md, /root/reference/PAPER.md line numbers "P:n"):
 *   For every pair of polygons p in P, q in Q whose minimum bounding rectangles
 *   overlap (the `&&` filter of Fig. 1(b), §2.2; the filter stage,
 *   §4.1), compute the exact pixel areas of intersection and union
 *   (PixelBox, §3, Alg. 1; union via |p u q| = |p| + |q| - |p n q|,
 *   P:75) and aggregate the Jaccard variant J' of Eq. (1) (§2.1).
 *
 * Geometry conventions (readings R1-R4):
 *   - A polygon is one ring of integer vertices with axis-parallel edges
 *     (§3.1), given as int32 (x, y) pixel-corner coordinates, implicitly
 *     closed (do not repeat the first vertex; a repeat is a harmless zero-length
 *     edge).  Either orientation.  The ring must be simple and hole-free
 *     (precondition, not checked).
 *   - Pixel (x, y) is the unit cell [x, x+1) x [y, y+1); it lies inside a
 *     polygon iff a ray cast from its center crosses the boundary an odd number
 *     of times.  Areas are pixel counts.
 *   - MBR = [min x, max x) x [min y, max y) (half-open); two MBRs overlap iff
 *     they share a pixel (touching MBRs do not pair; reading R4).
 *   - Limits: |coordinate| <= 2^30; every polygon's MBR is at most 65535 pixels
 *     wide and tall (edges are stored as 16-bit offsets); n_polygons < 2^31.
 *
 * Memory and ownership:
 *   - Every array pointer is a DEVICE pointer unless marked "host".  The caller
 *     allocates and owns every buffer, including derived per-polygon buffers and
 *     workspaces; the library allocates no device memory and keeps no state
 *     except a thread-local error slot.
 *   - All calls are stream-ordered on `stream` (a cudaStream_t; NULL = the
 *     legacy default stream).  Only sccg_filter_pairs synchronises (it returns
 *     the data-dependent pair count); the others return as soon as the work is
 *     enqueued.
 *
 * Errors: functions return an sccg_status.  Argument errors (SCCG_E_ARG,
 * SCCG_E_WORKSPACE) are detected on the host before anything is enqueued.
 * Data-dependent problems found on the device (non-rectilinear edge, range,
 * malformed offsets) set bits in a device status word (sccg_polyset.status,
 * sccg_sums.status); sccg_filter_pairs reads them after its sync and returns the
 * matching code.  sccg_last_error_index() reports the lowest offending polygon
 * index seen by the last failing call on this thread (-1 if none).
 */
#ifndef SCCG_H
#define SCCG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SCCG_API __attribute__((visibility("default")))
#else
#define SCCG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sccg_stream_t; /* == cudaStream_t */

typedef enum {
  SCCG_OK = 0,
  SCCG_E_ARG = 1,              /* null pointer, negative size, bad config, malformed offsets, < 4 vertices */
  SCCG_E_NOT_RECTILINEAR = 2,  /* a diagonal edge */
  SCCG_E_RANGE = 3,            /* |coord| > 2^30 or an MBR wider / taller than 65535 */
  SCCG_E_CAPACITY = 4,         /* output buffer too small; required size reported */
  SCCG_E_STACK = 5,            /* sampling-box stack overflow (internal bug) */
  SCCG_E_EMPTY = 6,            /* J' undefined: no pair with |p n q| != 0 (Eq. 1) */
  SCCG_E_CUDA = 7,             /* a CUDA runtime error (message in sccg_last_error_string) */
  SCCG_E_WORKSPACE = 8         /* workspace too small or misaligned */
} sccg_status;

/* status-word bits (device side) */
#define SCCG_STATUS_ARG (1u << 0)
#define SCCG_STATUS_NOT_RECTILINEAR (1u << 1)
#define SCCG_STATUS_RANGE (1u << 2)
#define SCCG_STATUS_STACK (1u << 3)
#define SCCG_STATUS_CAPACITY (1u << 4) /* sccg_pixelbox_async: the pair list overflowed its buffer; no pair processed */

/* One polygon set on the device: the caller's packed rings (inputs) plus the
 * per-polygon data sccg_prep derives from them (caller-allocated outputs; use
 * sccg_polyset_bind to carve them from one buffer of sccg_polyset_bytes). */
typedef struct {
  /* inputs */
  const int32_t* xy;      /* [n_vertices][2] interleaved x, y */
  const int64_t* offsets; /* [n_polygons + 1]; polygon i = vertices offsets[i] .. offsets[i+1]-1; offsets[0] = 0 */
  int64_t n_polygons;
  int64_t n_vertices;     /* == offsets[n_polygons] */
  /* derived by sccg_prep (§3.2 P:193 areas; MBRs for the filter) */
  int32_t* mbr;           /* [n_polygons][4] xlo, ylo, xhi, yhi (half-open pixel MBR) */
  int64_t* area;          /* [n_polygons] |p| (shoelace) */
  int32_t* ecount;        /* [n_polygons][2] vertical-edge count (bits 0-29) | raster flag (bit 30); the edge
                           * records' 16-bit rebase (internal layout) */
  uint64_t* edges;        /* [n_vertices] edge records (internal layout) */
  uint32_t* status;       /* [2] device: status bits (OR), lowest offending polygon (MIN) */
  void* stats;            /* [128 bytes] device: set statistics the join sizes its grid from (internal) */
} sccg_polyset;

/* Bytes of derived storage for a set (for sccg_polyset_bind). */
SCCG_API size_t sccg_polyset_bytes(int64_t n_polygons, int64_t n_vertices);

/* Point the derived fields of *set at sub-ranges of `buf` (device, 256-byte
 * aligned, at least sccg_polyset_bytes bytes).  Host-only, enqueues nothing. */
SCCG_API int sccg_polyset_bind(sccg_polyset* set, void* buf, size_t bytes);

/* Per-polygon prep: MBR, shoelace area (one term per
 * thread, summed), validation, and the edge records PixelBox reads.  Resets and
 * fills set->status.  validate = 1 checks rectilinearity, ranges, offsets. */
SCCG_API int sccg_prep(const sccg_polyset* set, int32_t validate, sccg_stream_t stream);

/* sccg_prep of `count` (1..4) independent sets in ONE launch: the sets' tiles
 * share one dynamically scheduled index space (one tail instead of one per
 * set).  `sets` is a host array of bound sets whose derived buffers are
 * disjoint; results are identical to calling sccg_prep on each.  Errors:
 * SCCG_E_ARG for count outside 1..4, a bad set, or shared derived buffers. */
SCCG_API int sccg_prep_sets(const sccg_polyset* sets, int32_t count, int32_t validate, sccg_stream_t stream);

/* The rings of a set in the packed transfer encoding (format 2, see sccg_decode_rect_packed below). */
typedef struct {
  const uint16_t* head;   /* [n_polygons] */
  const uint8_t* vlen;    /* [n_polygons], or NULL when no ring uses the variable-length class */
  const int16_t* start;   /* start stream */
  const uint16_t* units;  /* move units */
  const int64_t* block;   /* [ceil(n_polygons / SCCG_RECTP_BLOCK)][4] */
} sccg_rect_packed;

/* sccg_prep_sets with the rings arriving packed (rectilinear rings; the end-to-end path): each tile of
 * 128 rings is decoded straight into prep's shared-memory tile -- no separate decode kernel, no read of xy --
 * and written out, so on return (stream order) sets[i].offsets and sets[i].xy hold exactly what
 * sccg_decode_rect_packed would write (they are OUTPUT buffers here: device, writable, n_polygons + 1 int64 and
 * n_vertices int32 pairs, n_vertices the encoded total), and every derived field is what sccg_prep_sets
 * computes from them.  Device pointers; errors as sccg_prep_sets, and SCCG_E_ARG for a null or misaligned
 * encoding.  Asynchronous. */
SCCG_API int sccg_prep_sets_packed(const sccg_polyset* sets, const sccg_rect_packed* enc, int32_t count,
                                   int32_t validate, sccg_stream_t stream);

/* ---------------------------------------------------------------- filter */
/* Workspace bytes sccg_filter_pairs needs for sets of these sizes (the hashed
 * grid's bucket counters, 32 slots per bucket and an overflow pool, and the
 * probe tiles' pair buckets: about 700 bytes per Q polygon plus 8 KiB per
 * 128 P polygons).  The contents need no initialisation: every call clears
 * what it reads. */
SCCG_API size_t sccg_filter_workspace_bytes(int64_t n_p, int64_t n_q);

/* MBR-overlap join of two prepared sets by a hashed
 * uniform grid on the device (four kernels, no host round trip before the
 * count).  Writes the candidate pairs, unique and sorted by (p, q), as
 * pairs[k] = {p, q} (int32 [cap][2]) and sets *n_pairs_host (host) to their
 * count.  If cap < count (or pairs == NULL) SCCG_E_CAPACITY is returned with
 * *n_pairs_host = required count (the contents of pairs are then unspecified:
 * retry with a larger buffer).  Synchronises `stream` once (the count).  Also
 * returns the first data error recorded by sccg_prep in either set's status
 * word. */
SCCG_API int sccg_filter_pairs(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                      int64_t* n_pairs_host, void* workspace, size_t ws_bytes, sccg_stream_t stream);

/* As sccg_filter_pairs with CLOSED boxes: (p, q) pair when their MBRs share at
 * least a boundary point (touching MBRs included) -- the candidates of
 * sccg_touches.  Same workspace, errors and ordering. */
SCCG_API int sccg_filter_pairs_closed(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                                      int64_t* n_pairs_host, void* workspace, size_t ws_bytes,
                                      sccg_stream_t stream);

/* Asynchronous variant for device-resident pipelines (CUDA-graph capturable,
 * no host synchronisation): writes the candidate pairs when they fit in cap
 * (sorted by (p, q), as sccg_filter_pairs) and result_dev[0] = total pair
 * count, result_dev[1] = OR of both sets' sccg_prep status bits (device
 * int64[2]).  When result_dev[0] > cap some pairs were not written: read
 * result_dev after the stream synchronises and retry with a larger buffer. */
SCCG_API int sccg_filter_pairs_async(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                                     int64_t* result_dev, void* workspace, size_t ws_bytes, sccg_stream_t stream);

/* -------------------------------------------------------------- pixelbox */
/* Accumulated, order-independent integer totals (one NCCL int64 SUM merges
 * several GPUs bit-exactly).  Caller zeroes it once; each sccg_pixelbox call
 * adds to it (batching). */
typedef struct {
  int64_t n_pairs;       /* all pairs processed */
  int64_t n_nonzero;     /* pairs with |p n q| != 0 (the pairs Eq. 1 averages) */
  int64_t sum_inter;     /* sum |p n q| */
  int64_t sum_union;     /* sum |p u q| over pairs with |p n q| != 0 */
  int64_t sum_area_p;    /* sum |p| over all pairs (with multiplicity) */
  int64_t sum_area_q;    /* sum |q| over all pairs */
  int64_t ratio_limb[4]; /* sum of r = RN64(I/U) over I != 0, as an integer count of 2^-116 in 30-bit limbs */
  int64_t status;        /* OR of SCCG_STATUS_* bits seen */
} sccg_sums;

typedef struct {
  int32_t threshold; /* T: boxes with fewer pixels are pixelized (Alg. 1 l.22); 0 = default */
  int32_t mode;      /* 0 = PixelBox (Alg. 1: sampling boxes + pixelization over MBR(p) n MBR(q), union
                        from |p| + |q| - |p n q|); the paper's §5.2 baselines, which count the
                        union directly over the box of MBR(p) u MBR(q): 1 = PixelOnly (pixelization
                        only), 2 = PixelBox-NoSep (sampling boxes deciding both areas) */
  int32_t flags;     /* SCCG_FLAG_* bits; 0 = default */
  int32_t grid;      /* CTAs; 0 = default (resident CTAs per SM x SM count) */
  int64_t* counters; /* optional device int64[8] (NULL = off): see SCCG_CNT_* */
  uint32_t* hit_p;   /* optional device bitmaps, ceil(n/32) words, caller-zeroed: bit p (bit q) is set   */
  uint32_t* hit_q;   /* when polygon p of P (q of Q) has a pair with |p n q| != 0 (for missing counts)  */
} sccg_config;

/* flags: per-pair pixelization from edge records even where prep stored a ring's
 * raster (the paper's schedule, Alg. 1 l.24-25; results are identical) */
#define SCCG_FLAG_NO_RASTER 1
/* flags: every continuing sub-box of a split is pushed and processed on its own (Alg. 1 l.36-38 as
 * written).  By default a split whose sub-boxes are all below T and of which more than a quarter hover is
 * pixelized as one box instead (results are identical) */
#define SCCG_FLAG_PAPER_SPLIT 2

/* counters[] slots (accumulated; measurement builds only) */
#define SCCG_CNT_PIXELS 0      /* pixels classified by pixelization (each against both polygons) */
#define SCCG_CNT_ROWTESTS 1    /* (row segment x vertical edge) crossing tests */
#define SCCG_CNT_BOXES 2       /* sampling boxes classified (Lemma 1) */
#define SCCG_CNT_BOXEDGES 3    /* (sampling-box split x edge) classification steps */
#define SCCG_CNT_SPLITS 4      /* boxes split (SUBSAMPBOX calls) */
#define SCCG_CNT_PIXBOXES 5    /* boxes pixelized */
#define SCCG_CNT_ROOTPX 6      /* sum of root-box pixels |MBR(p) n MBR(q)| */

SCCG_API size_t sccg_pixelbox_workspace_bytes(int64_t n_pairs);

/* Optional extra workspace for the large path's per-pair edge index: any bytes
 * passed to sccg_pixelbox / sccg_pixelbox_async beyond
 * sccg_pixelbox_workspace_bytes(n) are used as an index pool.  A pair cut into
 * >= 4 region work items then has its rings' edges bucketed by region column
 * and row once (by the warp taking its first item), so its other items cull
 * only their buckets instead of both whole rings (Alg. 1 P:207-257 runs per
 * region; the areas are identical with or without the pool).  This returns a
 * pool size that indexes every large pair when each polygon is in about one
 * large pair: 8 bytes per vertex of both sets plus 16 MiB; pairs that do not
 * fit are processed unindexed.  n_vertices_* >= 0. */
SCCG_API size_t sccg_pixelbox_index_bytes(int64_t n_vertices_p, int64_t n_vertices_q);

/* PixelBox: for each pairs[k] = {p, q} (indices into the prepared
 * sets) write inter[k] = |p n q| and uni[k] = |p| + |q| - |p n q| (int64, input
 * order; either may be NULL to skip it) and add the batch's totals into *sums
 * (device).  Bit-identical results for every config, launch shape and GPU
 * count.  Asynchronous. */
SCCG_API int sccg_pixelbox(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                  int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg, void* workspace,
                  size_t ws_bytes, sccg_stream_t stream);

/* Asynchronous variant: processes pairs[0 .. result_dev[0]) where result_dev
 * is the device int64[2] written by sccg_filter_pairs_async, and ORs
 * result_dev[1] (prep status) into sums->status.  If result_dev[0] > cap (the
 * join overflowed the pair buffer, so the buffer is incomplete) no pair is
 * processed and SCCG_STATUS_CAPACITY is set in sums->status.  workspace as for
 * sccg_pixelbox_workspace_bytes(cap). */
SCCG_API int sccg_pixelbox_async(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs,
                                 const int64_t* result_dev, int64_t cap, int64_t* inter, int64_t* uni,
                                 sccg_sums* sums, const sccg_config* cfg, void* workspace, size_t ws_bytes,
                                 sccg_stream_t stream);

/* Missing polygons: the polygons of a set that appear in no pair with
 * |p n q| != 0, from a hit bitmap filled by sccg_pixelbox (config.hit_p /
 * hit_q).  Writes the count (n - set bits) to *missing_dev (device int64);
 * asynchronous. */
SCCG_API int sccg_count_missing(const uint32_t* hit, int64_t n, int64_t* missing_dev, sccg_stream_t stream);

/* ST_Touches (§3.4, reading R21 in DESIGN.md): touches[k] = 1
 * iff polygons p = pairs[k].x and q = pairs[k].y meet but their interiors do
 * not, i.e. inter[k] == 0 (the |p n q| sccg_pixelbox computed for the same
 * pairs; no common pixel) and some vertex of one ring lies on a (closed) edge
 * of the other -- the P:277 vertex-on-edge test; with no common pixel the
 * boundaries can only meet that way.  Candidates come from
 * sccg_filter_pairs_closed.  pairs: device int32 [n][2]; inter: device
 * int64 [n]; touches: device uint8 [n] (written).  Rings must be rectilinear
 * (sccg_prep validate).  Asynchronous; SCCG_E_ARG for null / negative /
 * misaligned arguments. */
SCCG_API int sccg_touches(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                          const int64_t* inter, uint8_t* touches, sccg_stream_t stream);

/* ST_Contains (§3.4: "computing the area of intersection and
 * testing whether it equals the area of the object being contained"): for each
 * pairs[k] = {p, q}, contains[k] bit 0 = p contains q (|p n q| == |q| > 0),
 * bit 1 = q contains p (|p n q| == |p| > 0), on the pixel model (R1: the pixel
 * set of the contained polygon is a subset of the other's).  inter: device
 * int64 [n] = the |p n q| sccg_pixelbox computed for the same pairs; pairs:
 * device int32 [n][2]; contains: device uint8 [n] (written; 0 for an
 * out-of-range index).  Sets must be prepared (areas).  Asynchronous; SCCG_E_ARG
 * for null / negative / misaligned arguments. */
SCCG_API int sccg_contains(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                           const int64_t* inter, uint8_t* contains, sccg_stream_t stream);

/* -------------------------------------------------------------- report */
/* Per-tile similarity report (SPEC S:343-346 SimilarityReport; Eq. 1 P:61 per
 * tile; missing polygons P:63).  The image is cut into a grid of ntx x nty tiles
 * of tile_w x tile_h pixels from (x0, y0); a polygon belongs to the tile holding
 * its MBR's lower-left corner (xlo, ylo) (clamped into the grid), a pair to the
 * tile of its p (reading R22). */
typedef struct {
  int32_t x0, y0;         /* grid origin */
  int32_t tile_w, tile_h; /* tile size in pixels (> 0) */
  int32_t ntx, nty;       /* tiles per row / column (> 0, ntx * nty < 2^31) */
} sccg_tiling;

/* One tile's entry: the pair totals of the tile's pairs in the sccg_sums
 * layout (sccg_jaccard on .sums gives the tile's J'), the tile's polygon counts
 * and its missing polygons (no pair with |p n q| != 0). */
typedef struct {
  sccg_sums sums;    /* status is 0 */
  int64_t n_poly_p;  /* polygons of P in the tile */
  int64_t n_poly_q;
  int64_t missing_p; /* ... of which appear in no pair with |p n q| != 0 */
  int64_t missing_q;
} sccg_tile_report;  /* 15 x int64 */

/* Accumulate the per-tile report of a pair batch into tiles[ntx * nty]
 * (device, caller-zeroed): pair totals from pairs / inter / uni (as written by
 * sccg_pixelbox for the same pairs), polygon and missing counts from the hit
 * bitmaps sccg_pixelbox filled (config.hit_p / hit_q; after every batch of the
 * image).  Polygon counts are added once per call: call it once per image with
 * all of the image's pairs (n_pairs may be 0).  Asynchronous; SCCG_E_ARG for
 * null / misaligned pointers or a bad tiling. */
SCCG_API int sccg_report(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                         const int64_t* inter, const int64_t* uni, const uint32_t* hit_p, const uint32_t* hit_q,
                         const sccg_tiling* tiling, sccg_tile_report* tiles, sccg_stream_t stream);

/* ---------------------------------------------------------------- jaccard */
/* J' of Eq. (1) from host-resident sums: the mean of r(p, q) over the
 * pairs with |p n q| != 0.  *pooled (nullable) = sum_inter / sum_union over the
 * same pairs.  Returns SCCG_E_EMPTY and NaN when n_nonzero == 0.  Sums that
 * carry status bits (a device-side error in any batch) are rejected: NaN and
 * the matching code (SCCG_E_ARG, _NOT_RECTILINEAR, _RANGE, _STACK, _CAPACITY,
 * checked in that order). */
SCCG_API int sccg_jaccard(const sccg_sums* sums_host, double* jprime, double* pooled);

/* Cross-GPU reduction of sums: sccg_sums_pack writes the
 * SCCG_REDUCE_WORDS int64 vector whose element-wise SUM over ranks (one NCCL
 * all-reduce) sccg_sums_unpack turns back into sums: words 0..9 are the ten
 * additive fields, words 10..25 status bit b (b < 16) as 0/1, so the reduced
 * status is the OR of the ranks' status words (a plain SUM of status would
 * carry bits into each other).  Device pointers, one single-warp kernel each;
 * asynchronous and graph-capturable.  SCCG_E_ARG for null / misaligned. */
#define SCCG_REDUCE_WORDS 26
SCCG_API int sccg_sums_pack(const sccg_sums* src, int64_t* vec, sccg_stream_t stream);
SCCG_API int sccg_sums_unpack(const int64_t* vec, sccg_sums* dst, sccg_stream_t stream);

/* Copy a sums block (88 bytes) from `src` (device) to `dst` with one single-warp kernel on `stream`, so a
 * step's result read-back needs no copy-engine round trip (it can sit inside a CUDA graph).  `dst` may be
 * device memory or page-locked host memory the device addresses through unified virtual addressing
 * (cudaHostAlloc / a pinned torch tensor); the stores are fenced system-wide, so the host sees them once an
 * event recorded after the call has completed.  Asynchronous.  Errors: SCCG_E_ARG for a null or
 * misaligned (not 8-byte) pointer. */
SCCG_API int sccg_sums_copy(const sccg_sums* src, sccg_sums* dst, sccg_stream_t stream);

/* Compact rectilinear rings, decoded on the device (an input encoding for the
 * host -> device transfer; the polygons are rectilinear, so a ring's
 * edges alternate between horizontal and vertical).  Ring i (offsets[i] ..
 * offsets[i + 1], as for sccg_polyset) starts at start[2i], start[2i + 1]; its
 * vertex k >= 1 moves from vertex k - 1 by move[offsets[i] - i + k - 1] (int16)
 * along x or y, alternating, the first move along y iff first_vertical[i] != 0.
 * Writes xy[2 * offsets[i] + 2k, +1] (int32) for every vertex: the plain layout
 * sccg_prep reads.  Device pointers; offsets must be valid (0 = offsets[0] <=
 * ... <= offsets[n]); n >= 0.  Asynchronous. */
SCCG_API int sccg_decode_rect(const int32_t* start, const int16_t* move, const uint8_t* first_vertical,
                              const int64_t* offsets, int64_t n, int32_t* xy, sccg_stream_t stream);

/* Packed rectilinear rings (format 2): the compact encoding above with each ring's moves at the narrowest of
 * four codings and no offsets on the wire (rectilinear rings; segmentation contours traced from a mask
 * move 1-3 pixels at a time, so a variable-length code takes ~2.2 bits per move instead of 16 + 64 per ring).
 * Rings are grouped in blocks of SCCG_RECTP_BLOCK consecutive rings (the last one partial).
 *   head[i]   uint16: vertex count V_i (bits 0-12, V_i <= 8191) | coding class w_i << 13 | (first edge vertical)
 *             << 15.  Vertex k >= 1 of ring i moves from vertex k - 1 by d along x or y, alternating, the first
 *             move along y iff head bit 15 is set; d != 0.
 *   units     uint16 stream: ring i's moves fill its units from unit u_i on (u_i = block[b][1] + the units of the
 *             block's earlier rings).  w = 0, 1, 2: fixed width, c = 4, 2, 1 moves per unit, move j of a unit in
 *             bits [j * b, (j + 1) * b), b = 16 / c, ceil((V_i - 1) / c) units; a 4- or 8-bit move is sign (top
 *             bit) and |d| - 1 (|d| <= 8 / 128); a 16-bit move is int16.  w = 3: variable length, vlen[i] units
 *             (<= 255): the units are one bit stream read from bit 0 of the first unit upward (unit j holds bits
 *             16j .. 16j + 15); move k - 1 is the symbol s = 2 (|d| - 1) + f, f = 1 iff the sign of d differs from
 *             that of the previous move along the same axis (for the first move along each axis: from +), coded as
 *             exp-Golomb LSB first: L zero bits, a one bit, then the L low bits of s + 1 (least significant
 *             first), L = floor(log2(s + 1)); |d| <= 127.
 *   vlen      uint8 [n]: units of ring i when w_i = 3 (read only then; may be NULL when no ring uses w = 3).
 *   start     int16 stream: ring j of block b starts at (x0 + start[s + 2j], y0 + start[s + 2j + 1]) when block b is
 *             narrow, at the int32 pair whose 16-bit halves are start[s + 4j .. s + 4j + 3] (x lo, x hi, y lo, y hi)
 *             when it is wide; s = block[b][2] & (2^62 - 1), wide = bit 62 of block[b][2], x0 = (int32) low half of
 *             block[b][3], y0 = (int32) high half.
 *   block     int64 [ceil(n / SCCG_RECTP_BLOCK)][4]: {offsets of the block's first ring, its u, s | wide << 62,
 *             (uint32) x0 | (uint64) (uint32) y0 << 32}.
 * Writes offsets[0 .. n] (int64, device; offsets[i + 1] - offsets[i] = V_i) and xy (int32 [offsets[n]][2]): exactly
 * the plain rings (the host encoder, paper_1208_0277_b200.encode_rect_packed, refuses rings it cannot express).
 * Device pointers; units / start 2-byte aligned, block / offsets / xy 8-byte aligned; n >= 0 (n = 0 writes
 * offsets[0] = 0).  Asynchronous.  Errors: SCCG_E_ARG for a negative n or a null / misaligned pointer. */
#define SCCG_RECTP_BLOCK 256
SCCG_API int sccg_decode_rect_packed(const uint16_t* head, const uint8_t* vlen, const int16_t* start,
                                     const uint16_t* units, const int64_t* block, int64_t n, int64_t* offsets,
                                     int32_t* xy, sccg_stream_t stream);

/* ------------------------------------------------------------------ misc */
SCCG_API const char* sccg_strerror(int code);
SCCG_API const char* sccg_last_error_string(void); /* thread-local detail of the last failure */
SCCG_API int64_t sccg_last_error_index(void);      /* thread-local; -1 if none */
SCCG_API int sccg_version(void);                   /* ABI version */

#ifdef __cplusplus
}
#endif
#endif /* SCCG_H */
