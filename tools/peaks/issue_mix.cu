// Can DFMA and integer/ALU instructions co-issue on B200?  Each warp runs
// 8 independent DFMA chains interleaved with NA independent integer ops per
// 8 DFMAs; prints cycles per (8 DFMA + NA ALU) group per SM sub-partition for
// W warps per sub-partition.  If ALU work hides under the 16 FP64-pipe cycles
// of 8 DFMAs the time stays flat up to NA ~ 8.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int NA>
__global__ void mix(double* out, int iters, double a, double b, unsigned m) {
  double x[8];
  unsigned y[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 16; ++i) y[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(a), "d"(b));
#pragma unroll
      for (int k = 0; k < NA / 8 + (i < NA % 8 ? 1 : 0); ++k) {
        const int j = (i * 2 + k) & 15;
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[j]) : "r"(m), "r"(y[(j + 1) & 15]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  unsigned t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t ^= y[i];
  if (s == 12345.678 || t == 0x12345) out[0] = s + t;
}

template <int NA>
int run(double* d, int nsm, int warps_per_sp, double mhz) {
  const int iters = 20000, threads = warps_per_sp * 4 * 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  mix<NA><<<nsm, threads>>>(d, iters, 0.999999, 1e-7, 0x5a5a5a5a);
  cudaEventRecord(e0);
  mix<NA><<<nsm, threads>>>(d, iters, 0.999999, 1e-7, 0x5a5a5a5a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * mhz * 1e6 / iters / warps_per_sp;  // per group per warp slot
  printf("W=%d NA=%2d  %.2f cycles per (8 DFMA + %d ALU) per sub-partition  -> FP64 pipe %.0f%%  IPC %.2f\n",
         warps_per_sp, NA, cyc, NA, 100.0 * 16 / cyc, (8 + NA) / cyc);
  return 0;
}

int main() {
  int nsm = 0, khz = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
  double* d; CK(cudaMalloc(&d, 64));
  const double mhz = khz / 1000.0;
  for (int w : {1, 2, 4}) {
    run<0>(d, nsm, w, mhz); run<4>(d, nsm, w, mhz); run<8>(d, nsm, w, mhz); run<12>(d, nsm, w, mhz);
    run<16>(d, nsm, w, mhz); run<24>(d, nsm, w, mhz);
  }
  return 0;
}
