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
#include "internal.cuh"

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

}  // namespace sccg
