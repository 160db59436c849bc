// api.cu -- the extern "C" boundary declared in include/sccg.h.
// Argument checking, workspace carving, the thread-local error slot, and
// sccg_jaccard (Eq. 1) on host-resident integer sums.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace sccg {

// NVTX range around each enqueueing entry point (header-only NVTX v3: a no-op
// unless a tool -- nsys, ncu --nvtx -- is attached), so a timeline or an ncu
// --nvtx-include filter can attribute kernels to the ABI call that issued them.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local char t_msg[256] = "";
static thread_local int64_t t_index = -1;

int set_error(int code, const char* msg, int64_t index) {
  snprintf(t_msg, sizeof(t_msg), "%s", msg ? msg : "");
  t_index = index;
  return code;
}

int check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return SCCG_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  return set_error(SCCG_E_CUDA, buf);
}

int decode_rect(const int32_t* start, const int16_t* move, const uint8_t* first_vertical, const int64_t* offsets,
                int64_t n, int32_t* xy, cudaStream_t stream);
int decode_rect_packed(const uint16_t* head, const uint8_t* vlen, const int16_t* start, const uint16_t* units,
                       const int64_t* block, int64_t n, int64_t* offsets, int32_t* xy, cudaStream_t stream);
size_t filter_ws_bytes(int64_t np, int64_t nq);
int filter_pairs(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap, int64_t* n_pairs_host,
                 void* ws, size_t ws_bytes, int closed, cudaStream_t stream);
int run_touches(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
                uint8_t* out, cudaStream_t stream);
size_t pixelbox_ws_bytes(int64_t n);
int run_contains(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
                 uint8_t* out, cudaStream_t stream);
int run_report(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
               const int64_t* uni, const uint32_t* hit_p, const uint32_t* hit_q, const sccg_tiling* tl,
               sccg_tile_report* tiles, cudaStream_t stream);
cudaError_t launch_sums_pack(const sccg_sums* src, int64_t* vec, cudaStream_t st);
cudaError_t launch_sums_unpack(const int64_t* vec, sccg_sums* dst, cudaStream_t st);
int count_missing(const uint32_t* hit, int64_t n, int64_t* out, cudaStream_t st);
int filter_pairs_async(const sccg_polyset* P, const sccg_polyset* Q, int32_t* pairs, int64_t cap,
                       int64_t* result_dev, void* ws, size_t ws_bytes, cudaStream_t stream);
int run_pixelbox(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n,
                 const int64_t* dev_result, int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg,
                 void* ws, size_t ws_bytes, cudaStream_t stream);

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

static int check_set(const sccg_polyset* s, bool need_derived, const char* name) {
  char buf[128];
  if (!s) {
    snprintf(buf, sizeof(buf), "%s: null sccg_polyset", name);
    return set_error(SCCG_E_ARG, buf);
  }
  if (s->n_polygons < 0 || s->n_vertices < 0 || s->n_polygons >= (int64_t(1) << 31)) {
    snprintf(buf, sizeof(buf), "%s: negative or too large size", name);
    return set_error(SCCG_E_ARG, buf);
  }
  if ((s->n_vertices > 0 && !s->xy) || !s->offsets) {
    snprintf(buf, sizeof(buf), "%s: null xy / offsets", name);
    return set_error(SCCG_E_ARG, buf);
  }
  if (!aligned(s->xy, 8) || !aligned(s->offsets, 8)) {
    snprintf(buf, sizeof(buf), "%s: xy / offsets must be 8-byte aligned", name);
    return set_error(SCCG_E_ARG, buf);
  }
  if (need_derived && (!s->mbr || !s->area || !s->ecount || (!s->edges && s->n_vertices > 0) || !s->status || !s->stats)) {
    snprintf(buf, sizeof(buf), "%s: derived buffers not bound (sccg_polyset_bind)", name);
    return set_error(SCCG_E_ARG, buf);
  }
  if (need_derived && (!aligned(s->mbr, 16) || !aligned(s->edges, 8) || !aligned(s->area, 8))) {
    snprintf(buf, sizeof(buf), "%s: derived buffers misaligned", name);
    return set_error(SCCG_E_ARG, buf);
  }
  return SCCG_OK;
}

static size_t polyset_layout(int64_t n, int64_t nv, Carve& cv, sccg_polyset* s) {
  int32_t* mbr = cv.take<int32_t>(4 * n);
  int64_t* area = cv.take<int64_t>(n);
  int32_t* ec = cv.take<int32_t>(2 * n);
  uint64_t* ed = cv.take<uint64_t>(nv);
  uint32_t* st = cv.take<uint32_t>(2);
  SetStats* ss = cv.take<SetStats>(1);
  if (s) {
    s->stats = ss;
    s->mbr = mbr;
    s->area = area;
    s->ecount = ec;
    s->edges = ed;
    s->status = st;
  }
  return cv.used;
}

}  // namespace sccg

using namespace sccg;

extern "C" {

int sccg_version(void) { return 1; }

const char* sccg_strerror(int code) {
  switch (code) {
    case SCCG_OK: return "ok";
    case SCCG_E_ARG: return "invalid argument";
    case SCCG_E_NOT_RECTILINEAR: return "polygon edge is not axis-parallel";
    case SCCG_E_RANGE: return "coordinate or polygon extent out of range";
    case SCCG_E_CAPACITY: return "output buffer too small";
    case SCCG_E_STACK: return "sampling-box stack overflow";
    case SCCG_E_EMPTY: return "no pair with non-zero intersection (J' undefined)";
    case SCCG_E_CUDA: return "CUDA error";
    case SCCG_E_WORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

const char* sccg_last_error_string(void) { return t_msg; }
int64_t sccg_last_error_index(void) { return t_index; }

size_t sccg_polyset_bytes(int64_t n_polygons, int64_t n_vertices) {
  if (n_polygons < 0 || n_vertices < 0) return 0;
  Carve cv{nullptr, ~size_t(0)};
  return polyset_layout(n_polygons, n_vertices, cv, nullptr) + 256;
}

int sccg_polyset_bind(sccg_polyset* set, void* buf, size_t bytes) {
  set_error(SCCG_OK, "", -1);
  if (!set || !buf) return set_error(SCCG_E_ARG, "sccg_polyset_bind: null argument");
  if (set->n_polygons < 0 || set->n_vertices < 0) return set_error(SCCG_E_ARG, "sccg_polyset_bind: negative size");
  if (!aligned(buf, 256)) return set_error(SCCG_E_WORKSPACE, "sccg_polyset_bind: buffer must be 256-byte aligned");
  Carve cv{reinterpret_cast<char*>(buf), bytes};
  polyset_layout(set->n_polygons, set->n_vertices, cv, set);
  if (!cv.ok) return set_error(SCCG_E_WORKSPACE, "sccg_polyset_bind: buffer smaller than sccg_polyset_bytes");
  return SCCG_OK;
}

int sccg_prep(const sccg_polyset* set, int32_t validate, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_prep");
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(set, true, "set")) return r;
  return check_cuda(launch_prep(&set, 1, validate, reinterpret_cast<cudaStream_t>(stream)), "sccg_prep");
}

int sccg_prep_sets(const sccg_polyset* sets, int32_t count, int32_t validate, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_prep_sets");
  set_error(SCCG_OK, "", -1);
  if (!sets || count < 1 || count > 4) return set_error(SCCG_E_ARG, "sccg_prep_sets: sets must hold 1..4 sets");
  const sccg_polyset* ptrs[4];
  for (int i = 0; i < count; i++) {
    if (int r = check_set(&sets[i], true, "sets[i]")) return r;
    for (int j = 0; j < i; j++)
      if (sets[j].stats == sets[i].stats || sets[j].status == sets[i].status)
        return set_error(SCCG_E_ARG, "sccg_prep_sets: sets must not share derived buffers");
    ptrs[i] = &sets[i];
  }
  return check_cuda(launch_prep(ptrs, count, validate, reinterpret_cast<cudaStream_t>(stream)), "sccg_prep_sets");
}

int sccg_prep_sets_packed(const sccg_polyset* sets, const sccg_rect_packed* enc, int32_t count, int32_t validate,
                          sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_prep_sets_packed");
  set_error(SCCG_OK, "", -1);
  if (!sets || !enc || count < 1 || count > 4)
    return set_error(SCCG_E_ARG, "sccg_prep_sets_packed: sets / enc must hold 1..4 sets");
  const sccg_polyset* ptrs[4];
  for (int i = 0; i < count; i++) {
    if (int r = check_set(&sets[i], true, "sets[i]")) return r;
    for (int j = 0; j < i; j++)
      if (sets[j].stats == sets[i].stats || sets[j].status == sets[i].status)
        return set_error(SCCG_E_ARG, "sccg_prep_sets_packed: sets must not share derived buffers");
    const sccg_rect_packed& e = enc[i];
    if (sets[i].n_polygons > 0 && (!e.head || !e.start || !e.block || !aligned(e.head, 2) || !aligned(e.start, 2) ||
                                   !aligned(e.units, 2) || !aligned(e.block, 8)))
      return set_error(SCCG_E_ARG, "sccg_prep_sets_packed: null or misaligned encoding", i);
    ptrs[i] = &sets[i];
  }
  return check_cuda(launch_prep(ptrs, count, validate, reinterpret_cast<cudaStream_t>(stream), enc),
                    "sccg_prep_sets_packed");
}

size_t sccg_filter_workspace_bytes(int64_t n_p, int64_t n_q) {
  if (n_p < 0 || n_q < 0) return 0;
  return filter_ws_bytes(n_p, n_q);
}

static int filter_checked(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                          int64_t* n_pairs_host, void* workspace, size_t ws_bytes, int closed, sccg_stream_t stream) {
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (!n_pairs_host) return set_error(SCCG_E_ARG, "n_pairs_host is null");
  if (cap < 0) return set_error(SCCG_E_ARG, "negative capacity");
  if (pairs && !aligned(pairs, 8)) return set_error(SCCG_E_ARG, "pairs must be 8-byte aligned");
  if (!workspace || !aligned(workspace, 256))
    return set_error(SCCG_E_WORKSPACE, "workspace must be non-null and 256-byte aligned");
  *n_pairs_host = 0;
  return filter_pairs(p, q, pairs, cap, n_pairs_host, workspace, ws_bytes, closed,
                      reinterpret_cast<cudaStream_t>(stream));
}

int sccg_filter_pairs(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                      int64_t* n_pairs_host, void* workspace, size_t ws_bytes, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_filter_pairs");
  return filter_checked(p, q, pairs, cap, n_pairs_host, workspace, ws_bytes, 0, stream);
}

int sccg_filter_pairs_closed(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                             int64_t* n_pairs_host, void* workspace, size_t ws_bytes, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_filter_pairs_closed");
  return filter_checked(p, q, pairs, cap, n_pairs_host, workspace, ws_bytes, 1, stream);
}

int sccg_touches(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                 const int64_t* inter, uint8_t* touches, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_touches");
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (n_pairs < 0) return set_error(SCCG_E_ARG, "negative pair count");
  if (n_pairs == 0) return SCCG_OK;
  if (!pairs || !aligned(pairs, 8)) return set_error(SCCG_E_ARG, "pairs must be a non-null 8-byte aligned device array");
  if (!inter || !aligned(inter, 8)) return set_error(SCCG_E_ARG, "inter must be a non-null aligned device int64 array");
  if (!touches) return set_error(SCCG_E_ARG, "touches is null");
  return run_touches(p, q, pairs, n_pairs, inter, touches, reinterpret_cast<cudaStream_t>(stream));
}

int sccg_contains(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                  const int64_t* inter, uint8_t* contains, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_contains");
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (n_pairs < 0) return set_error(SCCG_E_ARG, "negative pair count");
  if (n_pairs == 0) return SCCG_OK;
  if (!pairs || !aligned(pairs, 8)) return set_error(SCCG_E_ARG, "pairs must be a non-null 8-byte aligned device array");
  if (!inter || !aligned(inter, 8)) return set_error(SCCG_E_ARG, "inter must be a non-null aligned device int64 array");
  if (!contains) return set_error(SCCG_E_ARG, "contains is null");
  return run_contains(p, q, pairs, n_pairs, inter, contains, reinterpret_cast<cudaStream_t>(stream));
}

int sccg_report(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                const int64_t* inter, const int64_t* uni, const uint32_t* hit_p, const uint32_t* hit_q,
                const sccg_tiling* tiling, sccg_tile_report* tiles, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_report");
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (n_pairs < 0) return set_error(SCCG_E_ARG, "negative pair count");
  if (n_pairs > 0 && (!pairs || !inter || !uni)) return set_error(SCCG_E_ARG, "pairs / inter / uni is null");
  if (!aligned(pairs, 8) || !aligned(inter, 8) || !aligned(uni, 8)) return set_error(SCCG_E_ARG, "misaligned pointer");
  if ((p->n_polygons > 0 && !hit_p) || (q->n_polygons > 0 && !hit_q) || !aligned(hit_p, 4) || !aligned(hit_q, 4))
    return set_error(SCCG_E_ARG, "hit bitmaps must be non-null aligned device arrays");
  if (!tiling || !tiles || !aligned(tiles, 8)) return set_error(SCCG_E_ARG, "tiling / tiles is null or misaligned");
  if (tiling->tile_w <= 0 || tiling->tile_h <= 0 || tiling->ntx <= 0 || tiling->nty <= 0 ||
      (int64_t)tiling->ntx * tiling->nty >= (int64_t(1) << 31))
    return set_error(SCCG_E_ARG, "bad tiling (sizes and tile counts must be positive)");
  return run_report(p, q, pairs, n_pairs, inter, uni, hit_p, hit_q, tiling, tiles,
                    reinterpret_cast<cudaStream_t>(stream));
}

int sccg_sums_pack(const sccg_sums* src, int64_t* vec, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_sums_pack");
  set_error(SCCG_OK, "", -1);
  if (!src || !vec || !aligned(src, 8) || !aligned(vec, 8)) return set_error(SCCG_E_ARG, "sccg_sums_pack: null or misaligned pointer");
  return check_cuda(launch_sums_pack(src, vec, reinterpret_cast<cudaStream_t>(stream)), "sccg_sums_pack");
}

int sccg_sums_unpack(const int64_t* vec, sccg_sums* dst, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_sums_unpack");
  set_error(SCCG_OK, "", -1);
  if (!vec || !dst || !aligned(vec, 8) || !aligned(dst, 8)) return set_error(SCCG_E_ARG, "sccg_sums_unpack: null or misaligned pointer");
  return check_cuda(launch_sums_unpack(vec, dst, reinterpret_cast<cudaStream_t>(stream)), "sccg_sums_unpack");
}

int sccg_filter_pairs_async(const sccg_polyset* p, const sccg_polyset* q, int32_t* pairs, int64_t cap,
                            int64_t* result_dev, void* workspace, size_t ws_bytes, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_filter_pairs_async");
  set_error(SCCG_OK, "", -1);
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (!result_dev || !aligned(result_dev, 8)) return set_error(SCCG_E_ARG, "result_dev must be a non-null aligned device int64[2]");
  if (cap < 0) return set_error(SCCG_E_ARG, "negative capacity");
  if (pairs && !aligned(pairs, 8)) return set_error(SCCG_E_ARG, "pairs must be 8-byte aligned");
  if (!workspace || !aligned(workspace, 256))
    return set_error(SCCG_E_WORKSPACE, "workspace must be non-null and 256-byte aligned");
  return filter_pairs_async(p, q, pairs, cap, result_dev, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

size_t sccg_pixelbox_workspace_bytes(int64_t n_pairs) { return n_pairs < 0 ? 0 : pixelbox_ws_bytes(n_pairs); }

size_t sccg_pixelbox_index_bytes(int64_t n_vertices_p, int64_t n_vertices_q) {
  if (n_vertices_p < 0 || n_vertices_q < 0) return 0;
  return (size_t)8 * (size_t)(n_vertices_p + n_vertices_q) + ((size_t)1 << 24);
}

static int pixelbox_checks(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs,
                           int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg) {
  if (int r = check_set(p, true, "p")) return r;
  if (int r = check_set(q, true, "q")) return r;
  if (n_pairs < 0) return set_error(SCCG_E_ARG, "negative n_pairs");
  if (n_pairs > 0 && !pairs) return set_error(SCCG_E_ARG, "pairs is null");
  if (!sums) return set_error(SCCG_E_ARG, "sums is null");
  if (!aligned(sums, 8) || (pairs && !aligned(pairs, 8)) || (inter && !aligned(inter, 8)) || (uni && !aligned(uni, 8)))
    return set_error(SCCG_E_ARG, "misaligned pointer");
  if (cfg) {
    if (cfg->threshold < 0) return set_error(SCCG_E_ARG, "config.threshold < 0");
    if (cfg->flags & ~(SCCG_FLAG_NO_RASTER | SCCG_FLAG_PAPER_SPLIT))
      return set_error(SCCG_E_ARG, "config.flags: unknown bits");
    if (cfg->grid < 0) return set_error(SCCG_E_ARG, "config.grid < 0");
  }
  return SCCG_OK;
}

int sccg_pixelbox_async(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, const int64_t* result_dev,
                        int64_t cap, int64_t* inter, int64_t* uni, sccg_sums* sums, const sccg_config* cfg,
                        void* workspace, size_t ws_bytes, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_pixelbox_async");
  set_error(SCCG_OK, "", -1);
  if (!result_dev || !aligned(result_dev, 8)) return set_error(SCCG_E_ARG, "result_dev must be a non-null aligned device int64[2]");
  if (int r = pixelbox_checks(p, q, pairs, cap, inter, uni, sums, cfg)) return r;
  return run_pixelbox(p, q, pairs, cap, result_dev, inter, uni, sums, cfg, workspace, ws_bytes,
                      reinterpret_cast<cudaStream_t>(stream));
}

int sccg_pixelbox(const sccg_polyset* p, const sccg_polyset* q, const int32_t* pairs, int64_t n_pairs, int64_t* inter,
                  int64_t* uni, sccg_sums* sums, const sccg_config* cfg, void* workspace, size_t ws_bytes,
                  sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_pixelbox");
  set_error(SCCG_OK, "", -1);
  if (int r = pixelbox_checks(p, q, pairs, n_pairs, inter, uni, sums, cfg)) return r;
  return run_pixelbox(p, q, pairs, n_pairs, nullptr, inter, uni, sums, cfg, workspace, ws_bytes,
                      reinterpret_cast<cudaStream_t>(stream));
}

int sccg_count_missing(const uint32_t* hit, int64_t n, int64_t* missing_dev, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_count_missing");
  set_error(SCCG_OK, "", -1);
  if (n < 0 || !missing_dev || (n > 0 && !hit)) return set_error(SCCG_E_ARG, "sccg_count_missing: bad argument");
  if (!aligned(hit, 4) || !aligned(missing_dev, 8)) return set_error(SCCG_E_ARG, "sccg_count_missing: misaligned");
  return count_missing(hit, n, missing_dev, reinterpret_cast<cudaStream_t>(stream));
}

int sccg_decode_rect(const int32_t* start, const int16_t* move, const uint8_t* first_vertical,
                     const int64_t* offsets, int64_t n, int32_t* xy, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_decode_rect");
  set_error(SCCG_OK, "", -1);
  if (n < 0 || (n > 0 && (!start || !first_vertical || !offsets || !xy)) || !aligned(start, 8) || !aligned(xy, 8) ||
      !aligned(offsets, 8) || !aligned(move, 2))
    return set_error(SCCG_E_ARG, "sccg_decode_rect: bad size or null / misaligned pointer");
  return sccg::decode_rect(start, move, first_vertical, offsets, n, xy, reinterpret_cast<cudaStream_t>(stream));
}

int sccg_sums_copy(const sccg_sums* src, sccg_sums* dst, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_sums_copy");
  set_error(SCCG_OK, "", -1);
  if (!src || !dst || !aligned(src, 8) || !aligned(dst, 8)) return set_error(SCCG_E_ARG, "sccg_sums_copy: null or misaligned pointer");
  return check_cuda(launch_sums_copy(src, dst, reinterpret_cast<cudaStream_t>(stream)), "sccg_sums_copy");
}

int sccg_jaccard(const sccg_sums* s, double* jprime, double* pooled) {
  set_error(SCCG_OK, "", -1);
  if (!s || !jprime) return set_error(SCCG_E_ARG, "null argument");
  if (s->status) {  // a batch hit a device-side error: its totals are not the pairs' totals
    *jprime = NAN;
    if (pooled) *pooled = NAN;
    const int64_t b = s->status;
    const int code = (b & SCCG_STATUS_ARG) ? SCCG_E_ARG
                     : (b & SCCG_STATUS_NOT_RECTILINEAR) ? SCCG_E_NOT_RECTILINEAR
                     : (b & SCCG_STATUS_RANGE) ? SCCG_E_RANGE
                     : (b & SCCG_STATUS_STACK) ? SCCG_E_STACK
                     : (b & SCCG_STATUS_CAPACITY) ? SCCG_E_CAPACITY
                                                  : SCCG_E_ARG;
    char buf[96];
    snprintf(buf, sizeof(buf), "sums carry device status bits %#llx", (unsigned long long)b);
    return set_error(code, buf);
  }
  if (s->n_nonzero <= 0) {
    *jprime = NAN;
    if (pooled) *pooled = NAN;
    return set_error(SCCG_E_EMPTY, "no pair with |p n q| != 0");
  }
  // sum r = (L0 + L1 2^30 + L2 2^60 + L3 2^90) 2^-116; long double keeps 64
  // mantissa bits, so the one rounding to double dominates (reading R12).
  long double t = (long double)(uint64_t)s->ratio_limb[3];
  t = t * 1073741824.0L + (long double)(uint64_t)s->ratio_limb[2];
  t = t * 1073741824.0L + (long double)(uint64_t)s->ratio_limb[1];
  t = t * 1073741824.0L + (long double)(uint64_t)s->ratio_limb[0];
  t = ldexpl(t, -116);
  *jprime = (double)(t / (long double)s->n_nonzero);
  if (pooled) *pooled = (double)s->sum_inter / (double)s->sum_union;
  return SCCG_OK;
}

int sccg_decode_rect_packed(const uint16_t* head, const uint8_t* vlen, const int16_t* start, const uint16_t* units,
                            const int64_t* block, int64_t n, int64_t* offsets, int32_t* xy, sccg_stream_t stream) {
  NvtxRange nvtx_range("sccg_decode_rect_packed");
  set_error(SCCG_OK, "", -1);
  if (n < 0 || !offsets || (n > 0 && (!head || !start || !block || !xy)) || !aligned(head, 2) ||
      !aligned(start, 2) || !aligned(units, 2) || !aligned(block, 8) || !aligned(offsets, 8) || !aligned(xy, 8))
    return set_error(SCCG_E_ARG, "sccg_decode_rect_packed: bad size or null / misaligned pointer");
  return sccg::decode_rect_packed(head, vlen, start, units, block, n, offsets, xy,
                                  reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
