// predicates.cu -- other spatial predicates from the same kernels (SURVEY §8
// row f4, §3.4).
//
// ST_Touches.  P:277 sketches it as "no edge-to-edge crossing, no vertex of one
// polygon within the other, and at least one vertex of one polygon on the edge
// of the other".  Taken literally that calls two identical rings (or a ring
// and a contained ring sharing a side) touching although they overlap, so the
// interior test is taken from the areas instead (as ST_Contains is):
// reading R21 -- touches iff |p n q| == 0 (no common pixel, from PixelBox) and
// the boundaries meet.  With no common pixel two rectilinear boundaries can
// only meet where a vertex of one lies on a (closed) edge of the other (a
// proper crossing would put pixels of both on each side), which is the P:277
// vertex-on-edge test, done here warp per pair: lanes hold 32 vertices of one
// ring, the other ring's edges stream past as broadcast loads.
#include "internal.cuh"

namespace sccg {

constexpr int kTouchWarps = 8;

// Does any vertex of ring A (lane-parallel) lie on a closed edge of ring B?
// Vertices outside B's closed MBR are skipped without touching B's edges.
__device__ __forceinline__ bool vertex_on_edge(const int2* __restrict__ a, int64_t va, const int2* __restrict__ b,
                                               int64_t vb, const int4 mb) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = 0; i0 < va; i0 += 32) {
    const int64_t i = i0 + lane;
    int2 v = make_int2(0, 0);
    bool cand = false;
    if (i < va) {
      v = __ldg(a + i);
      cand = v.x >= mb.x && v.x <= mb.z && v.y >= mb.y && v.y <= mb.w;
    }
    if (!__any_sync(0xffffffffu, cand)) continue;
    bool on = false;
    int2 u = __ldg(b + vb - 1);  // edge (u, w): from the last vertex back to the first, then in order
    for (int64_t j = 0; j < vb; j++) {
      const int2 w = __ldg(b + j);
      if (cand) {
        if (u.x == w.x)
          on |= v.x == u.x && v.y >= min(u.y, w.y) && v.y <= max(u.y, w.y);
        else if (u.y == w.y)
          on |= v.y == u.y && v.x >= min(u.x, w.x) && v.x <= max(u.x, w.x);
      }
      u = w;
    }
    if (__any_sync(0xffffffffu, on)) return true;
  }
  return false;
}

__global__ void __launch_bounds__(kTouchWarps * 32)
    touches_kernel(const int2* __restrict__ xyp, const int64_t* __restrict__ offp, const int4* __restrict__ mbrp,
                   const int2* __restrict__ xyq, const int64_t* __restrict__ offq, const int4* __restrict__ mbrq,
                   int64_t np, int64_t nq, const int2* __restrict__ pairs, int64_t n,
                   const long long* __restrict__ inter, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * kTouchWarps;
  for (int64_t k = (int64_t)blockIdx.x * kTouchWarps + (threadIdx.x >> 5); k < n; k += nw) {  // warp per pair
    const int2 pq = pairs[k];
    bool t = false;
    if ((unsigned)pq.x < (unsigned long long)np && (unsigned)pq.y < (unsigned long long)nq && inter[k] == 0) {
      const int64_t bp = offp[pq.x], ep = offp[pq.x + 1], bq = offq[pq.y], eq = offq[pq.y + 1];
      const int4 mp = mbrp[pq.x], mq = mbrq[pq.y];
      const bool meet = mp.x <= mq.z && mq.x <= mp.z && mp.y <= mq.w && mq.y <= mp.w;  // closed MBRs
      if (meet && ep - bp >= 3 && eq - bq >= 3)
        t = vertex_on_edge(xyp + bp, ep - bp, xyq + bq, eq - bq, mq) ||
            vertex_on_edge(xyq + bq, eq - bq, xyp + bp, ep - bp, mp);
    }
    if (lane == 0) out[k] = t ? 1 : 0;
  }
}

int run_touches(const sccg_polyset* P, const sccg_polyset* Q, const int32_t* pairs, int64_t n, const int64_t* inter,
                uint8_t* out, cudaStream_t stream) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t blocks = (n + kTouchWarps - 1) / kTouchWarps;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  touches_kernel<<<(unsigned)blocks, kTouchWarps * 32, 0, stream>>>(
      reinterpret_cast<const int2*>(P->xy), P->offsets, reinterpret_cast<const int4*>(P->mbr),
      reinterpret_cast<const int2*>(Q->xy), Q->offsets, reinterpret_cast<const int4*>(Q->mbr), P->n_polygons,
      Q->n_polygons, reinterpret_cast<const int2*>(pairs), n, reinterpret_cast<const long long*>(inter), out);
  return check_cuda(cudaGetLastError(), "sccg_touches");
}

}  // namespace sccg
