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


// ------------------------------------------------------- packed (v2) format
// The same rings with the moves' bit width chosen per ring (4, 8 or 16 bits:
// nucleus contours traced from a mask move 1-3 pixels at a time, so 4 bits
// cover 99 % of the moves) and no offsets on the wire: ring i's vertex count
// travels in its 16-bit head and the device rebuilds the offsets by a block
// scan.  Starts travel as int16 deltas from the block's first start when the
// block allows it.  Layout: include/sccg.h (sccg_decode_rect_packed).
namespace {
constexpr int kRpBlock = SCCG_RECTP_BLOCK;  // rings per block (one CTA)
constexpr int kRpWarps = kRpBlock / 32;

__host__ __device__ __forceinline__ int rp_units(int m, int w) {  // 16-bit units holding m moves of width class w
  return w == 0 ? (m + 3) >> 2 : w == 1 ? (m + 1) >> 1 : m;
}

// One ring by one warp, C moves of BITS bits per 16-bit unit: a pass decodes
// 32 units (lane j unit j), lane-local prefix sums split into x and y (move i
// leads to vertex i + 1, which changes y iff (i + 1 odd) == vert), a warp scan
// of the lane totals, the pass's vertices staged in shared memory and stored
// coalesced.
template <int C, int BITS>
__device__ __forceinline__ void rp_ring(const unsigned short* __restrict__ up, int m, int vert, int cx, int cy,
                                        int2* __restrict__ dst, int2* stg) {
  const int lane = threadIdx.x & 31;
  const int nu = (m + C - 1) / C;
  for (int p0 = 0; p0 < nu; p0 += 32) {  // warp-uniform
    const int ui = p0 + lane;
    const unsigned u = ui < nu ? (unsigned)up[ui] : 0u;
    int px[C], py[C], sx = 0, sy = 0;
#pragma unroll
    for (int t = 0; t < C; t++) {
      int d;
      if (BITS == 16) {
        d = (int)(short)(u & 0xffffu);
      } else {
        const unsigned c = (u >> (BITS * t)) & ((1u << BITS) - 1u);
        const int mag = (int)(c & ((1u << (BITS - 1)) - 1u)) + 1;
        d = (c >> (BITS - 1)) ? -mag : mag;
      }
      const int i = ui * C + t;
      if (i >= m) d = 0;
      const bool ymove = ((i & 1) == 0) == (vert != 0);
      sx += ymove ? 0 : d;
      sy += ymove ? d : 0;
      px[t] = sx;
      py[t] = sy;
    }
    int ex = sx, ey = sy;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ex, o), b = __shfl_up_sync(0xffffffffu, ey, o);
      if (lane >= o) {
        ex += a;
        ey += b;
      }
    }
    const int tx = __shfl_sync(0xffffffffu, ex, 31), ty = __shfl_sync(0xffffffffu, ey, 31);
    ex += cx - sx;  // this lane's first move starts from here
    ey += cy - sy;
#pragma unroll
    for (int t = 0; t < C; t++) stg[lane * C + t] = make_int2(ex + px[t], ey + py[t]);
    __syncwarp();
    const int base = p0 * C, cnt = min(32 * C, m - base);
    for (int t = lane; t < cnt; t += 32) dst[base + t] = stg[t];
    __syncwarp();
    cx += tx;
    cy += ty;
  }
}
}  // namespace

__global__ void __launch_bounds__(kRpBlock) decode_rect_packed_kernel(const unsigned short* __restrict__ head,
                                                                      const short* __restrict__ start,
                                                                      const unsigned short* __restrict__ units,
                                                                      const long long* __restrict__ block, int64_t n,
                                                                      int64_t* __restrict__ off, int2* __restrict__ xy) {
  __shared__ int s_v[kRpBlock], s_u[kRpBlock], s_h[kRpBlock];
  __shared__ int2 s_s[kRpBlock];
  __shared__ int s_warp[2][kRpWarps];
  __shared__ int2 s_stage[kRpWarps][128];
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
  // ring head, start and unit count; block scan of (vertices, units)
  int V = 0, nu = 0, h = 0;
  int2 s0 = make_int2(0, 0);
  if (r < n) {
    h = head[r];
    V = h & 0x1fff;
    nu = rp_units(max(V - 1, 0), (h >> 13) & 3);
    const int j = threadIdx.x;
    if (wide) {
      const unsigned short* sp = reinterpret_cast<const unsigned short*>(start) + soff + 4 * j;
      s0 = make_int2((int)((unsigned)sp[0] | ((unsigned)sp[1] << 16)), (int)((unsigned)sp[2] | ((unsigned)sp[3] << 16)));
    } else {
      s0 = make_int2((int)(unsigned)(org & 0xffffffffll) + start[soff + 2 * j],
                     (int)(unsigned)((unsigned long long)org >> 32) + start[soff + 2 * j + 1]);
    }
  }
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
  __syncthreads();
  int bv = 0, bu = 0;
  for (int w = 0; w < warp; w++) {
    bv += s_warp[0][w];
    bu += s_warp[1][w];
  }
  s_v[threadIdx.x] = bv + xv - V;
  s_u[threadIdx.x] = bu + xu - nu;
  s_h[threadIdx.x] = h;
  s_s[threadIdx.x] = s0;
  if (r < n) {
    off[r] = vbase + bv + xv - V;
    if (r == n - 1) off[n] = vbase + bv + xv;
  }
  __syncthreads();
  // warp per ring: a pass decodes 32 units (up to 128 moves), lane j unit j;
  // lane-local prefix sums, a warp scan of the lane totals, vertices staged in
  // shared memory and stored coalesced
  const int nr = (int)min((int64_t)kRpBlock, n - b * kRpBlock);
  int2* stg = s_stage[warp];
  for (int j = warp; j < nr; j += kRpWarps) {
    const int hj = s_h[j], Vj = hj & 0x1fff, wj = (hj >> 13) & 3, vert = hj >> 15;
    const int m = max(Vj - 1, 0);
    const int64_t vo = vbase + s_v[j];
    const unsigned short* up = units + ubase + s_u[j];
    int cx = s_s[j].x, cy = s_s[j].y;
    if (Vj > 0 && lane == 0) xy[vo] = make_int2(cx, cy);
    int2* dst = xy + vo + 1;
    if (wj == 0)
      rp_ring<4, 4>(up, m, vert, cx, cy, dst, stg);
    else if (wj == 1)
      rp_ring<2, 8>(up, m, vert, cx, cy, dst, stg);
    else
      rp_ring<1, 16>(up, m, vert, cx, cy, dst, stg);
  }
}

int decode_rect_packed(const uint16_t* head, const int16_t* start, const uint16_t* units, const int64_t* block,
                       int64_t n, int64_t* offsets, int32_t* xy, cudaStream_t stream) {
  const int64_t nb = n > 0 ? (n + kRpBlock - 1) / kRpBlock : 1;
  launch_pdl(decode_rect_packed_kernel, dim3((unsigned)nb), dim3(kRpBlock), 0, stream,
             reinterpret_cast<const unsigned short*>(head), reinterpret_cast<const short*>(start),
             reinterpret_cast<const unsigned short*>(units), reinterpret_cast<const long long*>(block), n, offsets,
             reinterpret_cast<int2*>(xy));
  return check_cuda(cudaGetLastError(), "decode_rect_packed");
}

}  // namespace sccg
