// internal.cuh -- shared device helpers of the sm_100a PixelBox library.
// Not part of the ABI (see include/sccg.h).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sccg.h"

namespace sccg {

// Vertical-edge record (8 bytes, sccg_polyset.edges): edge x = const from
// ymin to ymax as three 16-bit fields c = x, lo = ymin, hi = ymax relative to
// an origin of the ring, mod 2^16 (decode_edge with ecount[i].y rebases them
// to the MBR lower-left corner: every field then fits 16 bits, MBR extent
// <= 65535).
// The records of polygon i occupy edges[off[i] .. off[i] + nv) in ring order
// (the rest of the polygon's slot is unspecified).  Horizontal edges are not
// stored: only sampling-box classification needs them, and it reads them from
// the ring itself.
// bit 48 of a vertical record: the ring traverses the edge upward (lo -> hi);
// decoders mask the three 16-bit fields and ignore it.
constexpr uint64_t kEdgeUp = 1ull << 48;
__host__ __device__ inline uint64_t pack_edge(uint32_t c, uint32_t lo, uint32_t hi) {
  return (uint64_t)c | ((uint64_t)lo << 16) | ((uint64_t)hi << 32);
}
__device__ __forceinline__ void unpack_edge(uint64_t r, int& c, int& lo, int& hi) {
  c = (int)(r & 0xffffu);
  lo = (int)((r >> 16) & 0xffffu);
  hi = (int)((r >> 32) & 0xffffu);
}

constexpr int kMaxExtent = 65535;
constexpr int64_t kMaxCoord = int64_t(1) << 30;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 32-bit shift left with PTX clamping: shift >= 32 gives 0.
__device__ __forceinline__ unsigned shl_clamp(unsigned a, unsigned s) {
  unsigned d;
  asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(s));
  return d;
}
// Mask of the pixels of a 32-pixel row word at or right of column k (k may be
// < 0 -> all, >= 32 -> none): the pixels an edge at x = k toggles when the
// crossing parity is counted toward -x (same parity as toward +x, because every
// row of a closed ring is crossed an even number of times).
__device__ __forceinline__ unsigned suffix_mask(int k) { return shl_clamp(0xffffffffu, (unsigned)max(k, 0)); }
// Low `n` bits (n in [0, 32]).
__device__ __forceinline__ unsigned low_bits(int n) { return ~shl_clamp(0xffffffffu, (unsigned)max(n, 0)); }

// ecount[i] = {nv | kRasterFlag when polygon i has a raster, o0}: nv = the
// vertical-edge count (bits 0-29); the raster is H = ymax - ylo 32-bit row
// words (bit x = pixel (xlo + x, ylo + r) inside) stored right after its
// vertical records, i.e. at (uint32*)(edges + off[i] + nv) (prep.cu).  The
// records' 16-bit fields are stored relative to some origin of the ring
// (its first vertex on the one-pass thread path, the MBR origin on the warp
// path) and o0 = (origin.x - xlo) | (origin.y - ylo) << 16 rebases them:
// decode_edge adds it mod 2^16 (every field of a valid ring lies in
// [0, 65535] relative to the MBR origin).
constexpr int kRasterFlag = 1 << 30;
constexpr int kNvMask = kRasterFlag - 1;
__device__ __forceinline__ void decode_edge(uint64_t r, unsigned o0, int& c, int& lo, int& hi) {
  c = (int)(((unsigned)r + o0) & 0xffffu);
  lo = (int)((((unsigned)(r >> 16) & 0xffffu) + (o0 >> 16)) & 0xffffu);
  hi = (int)((((unsigned)(r >> 32) & 0xffffu) + (o0 >> 16)) & 0xffffu);
}

// Per-set statistics written by sccg_prep (sccg_polyset.stats), read by the
// join's on-device grid selection: moments of the MBR extents over non-empty
// MBRs (w, h = width, height): sw = sum(w - 1), sh = sum(h - 1),
// swh = sum((w - 1)(h - 1)).  A 2^k grid cell count per MBR is at most
// ((w-1)/2^k + 2)((h-1)/2^k + 2) and about (1 + (w-1)/2^k)(1 + (h-1)/2^k).
struct SetStats {
  int32_t bounds[4];  // xmin, ymin, xmax, ymax over non-empty MBRs
  int32_t maxext[2];  // largest MBR width, height
  int32_t pad[2];
  unsigned long long nonempty, sw, sh, swh;
  unsigned long long reserved[8];
};
static_assert(sizeof(SetStats) == 128, "SetStats layout");

struct DevSet {
  const int2* xy;
  const int64_t* off;
  const int4* mbr;
  const int64_t* area;
  const int2* ecount;
  const uint64_t* edges;
};

inline DevSet dev_set(const sccg_polyset* s) {
  return DevSet{reinterpret_cast<const int2*>(s->xy), s->offsets, reinterpret_cast<const int4*>(s->mbr), s->area,
                reinterpret_cast<const int2*>(s->ecount), s->edges};
}

// Bump allocator over a caller workspace (256-byte aligned slices).
struct Carve {
  char* base;
  size_t cap, used = 0;
  bool ok = true;
  template <class T>
  T* take(size_t n) {
    size_t a = (used + 255) & ~size_t(255);
    size_t bytes = n * sizeof(T);
    if (a + bytes > cap) ok = false;
    used = a + bytes;
    return ok && base ? reinterpret_cast<T*>(base + a) : nullptr;
  }
};

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// be scheduled while its predecessor on the stream drains; it must execute
// pdl_wait() before touching anything the predecessor writes (the wait
// returns once the predecessor has completed and its writes are visible).
// pdl_trigger() lets the successor's CTAs launch early.  Both are no-ops
// without a programmatic dependency.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#ifdef SCCG_PDL_ACQUIRE
  // opt-in: acquire at GPU scope (MEMBAR + CCTL.IVALL in SASS) invalidates this
  // SM's L1 after the wait.  Not needed with late triggers (a kernel's CTAs
  // start only after its predecessor passed its own wait) plus L2 loads of the
  // control words (ld_coherent); measured 3 % slower on C2 (0.308 vs 0.299 ms)
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
#endif
}

// Control words a predecessor kernel of a PDL chain wrote (a grid
// descriptor, a device-side count) are read with L1-bypassing loads after
// pdl_wait(): a CTA launched early may otherwise see a stale L1 / read-only
// cache line of a recycled address (measured on the join's grid descriptor).
__device__ __forceinline__ long long ld_coherent(const long long* p) { return __ldcg(p); }  // ld.global.cg: L2

// Where a kernel lets its successor launch.  Early (SCCG_PDL_LATE=0, the
// round-1 order): trigger at entry, so the successor's CTAs -- and, since
// they trigger at entry too, every later kernel's -- can become resident
// while this one still runs, holding registers and warp slots as they wait.
// Late (default): a kernel triggers after its own wait, and the two big
// persistent kernels (prep, the small PixelBox kernel) only once their work
// queue is drained, so at most the next kernel waits resident.
#ifndef SCCG_PDL_LATE
#define SCCG_PDL_LATE 1
#endif
__device__ __forceinline__ void pdl_entry() {
  if (!SCCG_PDL_LATE) pdl_trigger();
  pdl_wait();
  if (SCCG_PDL_LATE) pdl_trigger();
}
// for kernels that trigger themselves once their main loop is done
__device__ __forceinline__ void pdl_entry_deferred() {
  if (!SCCG_PDL_LATE) pdl_trigger();
  pdl_wait();
}
__device__ __forceinline__ void pdl_done() {
  if (SCCG_PDL_LATE) pdl_trigger();
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef SCCG_NO_PDL  // ablation build (scripts/fig9.py): plain stream-ordered launches
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// error slot (api.cu)
int set_error(int code, const char* msg, int64_t index = -1);
int check_cuda(cudaError_t e, const char* where);

// launchers
cudaError_t launch_prep(const sccg_polyset* const* sets, int count, int validate, cudaStream_t st,
                        const sccg_rect_packed* pk = nullptr);
cudaError_t launch_sums_copy(const sccg_sums* src, sccg_sums* dst, cudaStream_t st);

}  // namespace sccg
