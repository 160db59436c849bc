// packed_decode.cuh -- one ring of the packed rectilinear encoding (format 2,
// include/sccg.h sccg_decode_rect_packed) walked by one thread; shared by the
// decode kernel (decode.cu) and prep's packed mode (prep.cu).  Not ABI.
#pragma once
#include "internal.cuh"

namespace sccg {

constexpr int kRpBlock = SCCG_RECTP_BLOCK;  // rings per block

__host__ __device__ __forceinline__ int rp_units(int m, int w) {  // 16-bit units holding m moves of width class w
  return w == 0 ? (m + 3) >> 2 : w == 1 ? (m + 1) >> 1 : m;
}

// Ring of V >= 1 vertices, head bits (class w, first-vertical bit vert), its
// move units at `up`, start (x, y): writes dst[0 .. V).  Vertex k >= 1 changes
// y iff (k odd) == vert.
__device__ __forceinline__ void rp_walk_ring(const unsigned short* __restrict__ up, int V, int w, int vert, int x,
                                             int y, int2* __restrict__ dst) {
  dst[0] = make_int2(x, y);
  if (w == 3) {
    // variable-length moves: symbol s = 2 (|d| - 1) + flip, flip = the sign
    // differs from the previous move on the same axis (the first one on each
    // axis: from +), exp-Golomb coded LSB-first -- L zero bits, a one, the
    // L low bits of s + 1; bits refilled 16 at a time into a 32-bit window
    // (a code is at most 15 bits: |d| <= 127)
    unsigned b = 0u;  // bit window (32-bit: a code is <= 15 bits, refills of 16 keep it >= 16 bits)
    int nb = 0, ui = 0;
    int sa = 0, sb = 0;  // sign state of the axis of the even / odd moves
    int pa = vert ? y : x, pb = vert ? x : y;  // position along the axis of the even / odd moves
    auto next = [&](int& sgn) {  // one symbol -> the signed move
      if (nb < 16) {
        b |= (unsigned)up[ui] << nb;
        ui++;
        nb += 16;
      }
      const int L = __ffs((int)b) - 1;
      const unsigned t = b >> (L + 1);
      const int sym = (int)((1u << L) | (t & ((1u << L) - 1u))) - 1;
      b = t >> L;
      nb -= 2 * L + 1;
      sgn ^= sym & 1;
      const int mag = (sym >> 1) + 1;
      return sgn ? -mag : mag;
    };
    auto put = [&](int k) { dst[k] = vert ? make_int2(pb, pa) : make_int2(pa, pb); };
    int k = 1;
    for (; k + 2 <= V; k += 2) {  // moves k - 1 (even) and k (odd): the axis pattern is static
      pa += next(sa);
      put(k);
      pb += next(sb);
      put(k + 1);
    }
    if (k < V) {
      pa += next(sa);
      put(k);
    }
  } else {
    const int lc = w == 0 ? 2 : w == 1 ? 1 : 0;  // log2(moves per unit)
    const int bits = 16 >> lc;
    const unsigned mask = bits == 16 ? 0xffffu : (1u << bits) - 1u, mmag = mask >> 1;
    const int cm = (1 << lc) - 1;
    unsigned cur = 0u;
    for (int k = 1; k < V; k++) {
      const int mi = k - 1;
      if ((mi & cm) == 0) cur = up[mi >> lc];  // a unit is read once (predicated, not per move)
      const unsigned code = (cur >> ((mi & cm) * bits)) & mask;
      const int mag = (int)(code & mmag) + 1;
      const int d = bits == 16 ? (int)(short)code : ((code > mmag) ? -mag : mag);
      const bool ymove = (k & 1) == vert;
      x += ymove ? 0 : d;
      y += ymove ? d : 0;
      dst[k] = make_int2(x, y);
    }
  }
}

}  // namespace sccg
