// decode.cu -- compact rectilinear rings for the host->device transfer.
//
// A rectilinear ring alternates horizontal and vertical edges (the
// segmented polygons are rectilinear), so after its first vertex each vertex
// differs from the previous one in exactly one coordinate, and which one
// alternates.  The compact form keeps the first vertex (int32 x, y), one bit
// for the axis of the first edge, and one int16 signed move per further
// vertex: 2 bytes per vertex instead of 8, so a PCIe-bound end-to-end step
// moves a quarter of the vertex bytes.  (Encoder: paper_1208_0277_b200.
// encode_rect; rings with a zero-length or collinear edge, or a move beyond
// int16, are not encodable and travel as plain xy.)  The decode writes the
// ring's vertices exactly (integer prefix sums): decode(encode(xy)) == xy.
#include "packed_decode.cuh"

namespace sccg {

// Warp per ring, 32 vertices at a time: lane j holds vertex k = k0 + j; its x
// is the start x plus every x-move up to k (moves 1, 3, 5, ... when the first
// edge is horizontal), its y likewise with the other parity -- two inclusive
// warp scans, carried across chunks.  Coalesced int2 stores.
__global__ void decode_rect_kernel(const int2* __restrict__ start, const short* __restrict__ move,
                                   const unsigned char* __restrict__ first_vertical, const int64_t* __restrict__ off,
                                   int64_t n, int2* __restrict__ xy) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t b = off[r], e = off[r + 1];
    const int64_t mb = b - r;  // ring r's moves: vertices 1 .. V-1 of ring r are moves mb .. mb + V - 2
    const int2 s0 = start[r];
    const int vert = first_vertical[r] ? 1 : 0;  // move k (k >= 1) changes y iff (k odd) == vert
    int cx = s0.x, cy = s0.y;
    for (int64_t k0 = 0; k0 < e - b; k0 += 32) {  // warp-uniform
      const int64_t k = k0 + lane;
      int dx = 0, dy = 0;
      if (k >= 1 && k < e - b) {
        const int d = move[mb + k - 1];
        if (((int)(k & 1) == 1) == (vert == 1)) dy = d;
        else dx = d;
      }
      for (int o = 1; o < 32; o <<= 1) {
        const int ux = __shfl_up_sync(0xffffffffu, dx, o), uy = __shfl_up_sync(0xffffffffu, dy, o);
        if (lane >= o) {
          dx += ux;
          dy += uy;
        }
      }
      if (k < e - b) xy[b + k] = make_int2(cx + dx, cy + dy);
      cx += __shfl_sync(0xffffffffu, dx, 31);
      cy += __shfl_sync(0xffffffffu, dy, 31);
    }
  }
}

int decode_rect(const int32_t* start, const int16_t* move, const uint8_t* first_vertical, const int64_t* offsets,
                int64_t n, int32_t* xy, cudaStream_t stream) {
  if (n <= 0) return SCCG_OK;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t blocks = (n * 32 + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  launch_pdl(decode_rect_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, reinterpret_cast<const int2*>(start),
             reinterpret_cast<const short*>(move), first_vertical, offsets, n, reinterpret_cast<int2*>(xy));
  return check_cuda(cudaGetLastError(), "decode_rect");
}


// ------------------------------------------------------- packed (v2) format
// The same rings with the moves' bit width chosen per ring (4, 8 or 16 bits:
// nucleus contours traced from a mask move 1-3 pixels at a time, so 4 bits
// cover 99 % of the moves) and no offsets on the wire: ring i's vertex count
// travels in its 16-bit head and the device rebuilds the offsets by a block
// scan.  Starts travel as int16 deltas from the block's first start when the
// block allows it.  Layout: include/sccg.h (sccg_decode_rect_packed).
namespace {
constexpr int kRpWarps = kRpBlock / 32;

// Staging capacity: a block's vertices (thread per ring, ~8.7 k vertices for
// 256 nucleus rings) are assembled in shared memory and leave by coalesced
// stores; its move units arrive by one coalesced pass.  Rings past either
// capacity (blocks of very long rings) read / write global memory directly.
constexpr int kRpStage = 7168;  // int2 vertices (56 KB)
constexpr int kRpUnits = 4096;  // 16-bit units (8 KB)
constexpr size_t kRpSmem = kRpStage * sizeof(int2) + kRpUnits * sizeof(unsigned short);
}  // namespace

// CTA per block of kRpBlock rings, thread per ring: heads -> block scan of
// (vertices, units) -> the block's offsets; units staged; each thread walks
// its ring's moves (vertex k >= 1 changes y iff (k odd) == the first-vertical
// bit; the width class selects 4, 2 or 1 moves per unit) writing vertices into
// the staged block; the staged range is stored coalesced.
__global__ void __launch_bounds__(kRpBlock) decode_rect_packed_kernel(const unsigned short* __restrict__ head,
                                                                      const unsigned char* __restrict__ vlen,
                                                                      const short* __restrict__ start,
                                                                      const unsigned short* __restrict__ units,
                                                                      const long long* __restrict__ block, int64_t n,
                                                                      int64_t* __restrict__ off, int2* __restrict__ xy) {
  extern __shared__ __align__(16) unsigned char rp_smem[];
  int2* s_stage = reinterpret_cast<int2*>(rp_smem);
  unsigned short* s_units = reinterpret_cast<unsigned short*>(rp_smem + kRpStage * sizeof(int2));
  __shared__ int s_warp[2][kRpWarps];
  __shared__ int s_lim;
  pdl_entry();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = blockIdx.x, r = b * kRpBlock + threadIdx.x;
  if (n == 0) {
    if (threadIdx.x == 0) off[0] = 0;
    return;
  }
  const long long vbase = block[4 * b], ubase = block[4 * b + 1], sw = block[4 * b + 2], org = block[4 * b + 3];
  const bool wide = (sw >> 62) & 1;
  const long long soff = sw & ((1ll << 62) - 1);
  int V = 0, nu = 0, h = 0, x = 0, y = 0;
  if (r < n) {
    h = head[r];
    V = h & 0x1fff;
    const int w = (h >> 13) & 3;
    nu = w == 3 ? (int)vlen[r] : rp_units(max(V - 1, 0), w);
    const int j = threadIdx.x;
    if (wide) {
      const unsigned short* sp = reinterpret_cast<const unsigned short*>(start) + soff + 4 * j;
      x = (int)((unsigned)sp[0] | ((unsigned)sp[1] << 16));
      y = (int)((unsigned)sp[2] | ((unsigned)sp[3] << 16));
    } else {
      x = (int)(unsigned)(org & 0xffffffffll) + start[soff + 2 * j];
      y = (int)(unsigned)((unsigned long long)org >> 32) + start[soff + 2 * j + 1];
    }
  }
  // block scan of (vertices, units)
  int xv = V, xu = nu;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, xv, o), c = __shfl_up_sync(0xffffffffu, xu, o);
    if (lane >= o) {
      xv += a;
      xu += c;
    }
  }
  if (lane == 31) {
    s_warp[0][warp] = xv;
    s_warp[1][warp] = xu;
  }
  if (threadIdx.x == 0) s_lim = INT_MAX;
  __syncthreads();
  int bv = 0, bu = 0, tv = 0, tu = 0;
  for (int w = 0; w < kRpWarps; w++) {
    bv += w < warp ? s_warp[0][w] : 0;
    bu += w < warp ? s_warp[1][w] : 0;
    tv += s_warp[0][w];
    tu += s_warp[1][w];
  }
  const int v0 = bv + xv - V, u0 = bu + xu - nu;  // this ring's vertex / unit offsets in the block
  if (r < n) {
    off[r] = vbase + v0;
    if (r == n - 1) off[n] = vbase + v0 + V;
  }
  const bool staged = v0 + V <= kRpStage;
  if (r < n && !staged) atomicMin(&s_lim, v0);
  // the block's units, coalesced
  const int nus = min(tu, kRpUnits);
  for (int i = threadIdx.x; i < nus; i += kRpBlock) s_units[i] = units[ubase + i];
  __syncthreads();
  if (r < n && V > 0) {
    const int w = (h >> 13) & 3, vert = h >> 15;
    const unsigned short* up = u0 + nu <= kRpUnits ? s_units + u0 : units + ubase + u0;
    int2* dst = staged ? s_stage + v0 : xy + vbase + v0;
    rp_walk_ring(up, V, w, vert, x, y, dst);
  }
  __syncthreads();
  const int lim = min(tv, s_lim);
  for (int i = threadIdx.x; i < lim; i += kRpBlock) xy[vbase + i] = s_stage[i];
}

int decode_rect_packed(const uint16_t* head, const uint8_t* vlen, const int16_t* start, const uint16_t* units,
                       const int64_t* block, int64_t n, int64_t* offsets, int32_t* xy, cudaStream_t stream) {
  const int64_t nb = n > 0 ? (n + kRpBlock - 1) / kRpBlock : 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_rect_packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRpSmem);
    attr = true;
  }
  launch_pdl(decode_rect_packed_kernel, dim3((unsigned)nb), dim3(kRpBlock), kRpSmem, stream,
             reinterpret_cast<const unsigned short*>(head), vlen, reinterpret_cast<const short*>(start),
             reinterpret_cast<const unsigned short*>(units), reinterpret_cast<const long long*>(block), n, offsets,
             reinterpret_cast<int2*>(xy));
  return check_cuda(cudaGetLastError(), "decode_rect_packed");
}

}  // namespace sccg
