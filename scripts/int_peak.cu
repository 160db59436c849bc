// int_peak.cu -- integer-issue microbenchmark (SURVEY §7.1 step 1, §8(d)
// "Roofline": the denominator of "vs int-issue peak").
//
// Each thread runs 8 independent loop-carried chains of one instruction class
// (inline PTX; the SASS per step was checked with cuobjdump -sass), so the rate is
// limited by the pipe, not by latency.  The rate is reported as warp
// instructions per SM cycle (SM cycles from %clock64 per CTA, kernel span =
// the longest CTA) and per second (CUDA events).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
//   ./int_peak  -> one JSON object on stdout
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

constexpr int kChains = 8;
constexpr int kUnroll = 16;

// op classes (per chain step; instructions per step in kInstPerStep)
enum Op { LOP3 = 0, IADD3, IMAD, LOP3_IMAD, ISETP_SEL, POPC, SHF, ROWTEST, NOPS };
static const char* kName[NOPS] = {"lop3", "iadd3", "imad", "lop3+imad", "isetp+sel", "popc", "shf", "rowtest"};
static const int kInstPerStep[NOPS] = {1, 1, 1, 2, 2, 2, 1, 2};  // SASS per step (checked: ROWTEST = LOP3 -> P, @P LOP3)
static const char* kPipe[NOPS] = {"alu", "alu", "fma", "alu+fma", "alu", "popc+alu", "alu", "alu"};

template <int OP>
__device__ __forceinline__ void step(unsigned& a, unsigned b, unsigned c) {
  if constexpr (OP == LOP3) {
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
  } else if constexpr (OP == IADD3) {
    asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a) : "r"(b), "r"(c));  // fused into one IADD3
  } else if constexpr (OP == IMAD) {
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  } else if constexpr (OP == LOP3_IMAD) {
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;\n\tmad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
  } else if constexpr (OP == ISETP_SEL) {
    asm volatile("{ .reg .pred p; setp.gt.u32 p, %0, %1; selp.b32 %0, %2, %0, p; }" : "+r"(a) : "r"(b), "r"(c));
  } else if constexpr (OP == POPC) {
    asm volatile("{ .reg .b32 t; popc.b32 t, %0; xor.b32 %0, t, %1; }" : "+r"(a) : "r"(b));
  } else if constexpr (OP == SHF) {
    asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a) : "r"(b));
  } else if constexpr (OP == ROWTEST) {
    // the PixelBox crossing-test shape: row-bit AND, compare, predicated XOR
    asm volatile("{ .reg .pred p; .reg .b32 t; and.b32 t, %0, %1; setp.ne.u32 p, t, 0; @p xor.b32 %0, %0, %2; }"
                 : "+r"(a) : "r"(b), "r"(c));
  }
}

template <int OP>
__global__ void chains(unsigned* out, long long* span, int iters, unsigned seed) {
  unsigned r[kChains];
#pragma unroll
  for (int k = 0; k < kChains; k++) r[k] = seed * (threadIdx.x + 1) + k;
  const unsigned b = seed ^ threadIdx.x, c = seed + blockIdx.x;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
#pragma unroll
      for (int k = 0; k < kChains; k++) step<OP>(r[k], b, c);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  unsigned x = 0;
#pragma unroll
  for (int k = 0; k < kChains; k++) x ^= r[k];
  if (x == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = x;  // keeps the chains live
  if (threadIdx.x == 0) span[blockIdx.x] = t1 - t0;
}

template <int OP>
int run(int sms, int warps_per_sm, int iters, double* inst_per_clk, double* inst_per_s, double* mhz) {
  const int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
  const int blocks_per_sm = warps_per_sm * 32 / threads;
  const int blocks = sms * blocks_per_sm;
  unsigned* out;
  long long* span;
  CK(cudaMalloc(&out, (size_t)blocks * threads * 4));
  CK(cudaMalloc(&span, blocks * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<OP><<<blocks, threads>>>(out, span, iters / 8, 1u);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  chains<OP><<<blocks, threads>>>(out, span, iters, 3u);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  CK(cudaMemcpy(h, span, blocks * 8, cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  delete[] h;
  const double warp_inst = (double)blocks * threads / 32 * iters * kUnroll * kChains * kInstPerStep[OP];
  *inst_per_clk = warp_inst / sms / (double)mx;
  *inst_per_s = warp_inst / (ms * 1e-3);
  *mhz = (double)mx / (ms * 1e-3) / 1e6;  // approximate (includes launch overhead)
  cudaFree(out);
  cudaFree(span);
  return 0;
}

template <int OP>
int sweep(int sms, bool& first) {
  const int warps[] = {8, 16, 32, 64};
  for (int w : warps) {
    double ipc = 0, ips = 0, mhz = 0;
    if (run<OP>(sms, w, 4096, &ipc, &ips, &mhz)) return 1;
    printf("%s\n    {\"op\": \"%s\", \"pipe\": \"%s\", \"inst_per_step\": %d, \"warps_per_sm\": %d, "
           "\"warp_inst_per_clk_per_sm\": %.4f, \"warp_inst_per_s\": %.4e, \"sm_mhz_est\": %.0f}",
           first ? "" : ",", kName[OP], kPipe[OP], kInstPerStep[OP], w, ipc, ips, mhz);
    first = false;
  }
  return 0;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_rate_mhz\": %.0f, \"chains_per_thread\": %d, \"results\": [",
         prop.name, sms, clk_khz / 1e3, kChains);
  bool first = true;
  if (sweep<LOP3>(sms, first) || sweep<IADD3>(sms, first) || sweep<IMAD>(sms, first) ||
      sweep<LOP3_IMAD>(sms, first) || sweep<ISETP_SEL>(sms, first) || sweep<POPC>(sms, first) ||
      sweep<SHF>(sms, first) || sweep<ROWTEST>(sms, first))
    return 1;
  printf("\n]}\n");
  return 0;
}
