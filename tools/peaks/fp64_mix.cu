// Do DMMA (mma.sync m8n8k4 f64) and DFMA share the FP64 units on B200?
// Runs DFMA alone, DMMA alone, and both at once (warps split inside each
// CTA, and both streams interleaved inside every warp); prints one JSON line
// of TFLOP/s.  If the mixed rates add up, the two pipes are separate.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void dfma8(double (&x)[8], double a, double b) {
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
}
__device__ __forceinline__ void dmma4(double (&c)[4][2], double a, double b) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
}

// mode 0: DFMA only; 1: DMMA only; 2: even warps DFMA, odd warps DMMA;
// 3: every warp alternates one DMMA group and `ratio` DFMA groups
__global__ void mix(double* out, int iters, int mode, int ratio, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double c[4][2] = {};
  const int warp = threadIdx.x >> 5;
  const bool do_f = mode == 0 || mode == 3 || (mode == 2 && !(warp & 1));
  const bool do_m = mode == 1 || mode == 3 || (mode == 2 && (warp & 1));
  for (int it = 0; it < iters; ++it) {
    if (do_m) dmma4(c, a, b);
    if (do_f)
      for (int r = 0; r < (mode == 3 ? ratio : 1); ++r) dfma8(x, a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int nsm = 0;
  CK(cudaSetDevice(0));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double* d;
  CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 4, threads = 256, iters = 20000;
  auto run = [&](int mode, int ratio) {
    for (int i = 0; i < 2; ++i) mix<<<blocks, threads>>>(d, iters, mode, ratio, 0.999999, 1e-7);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) mix<<<blocks, threads>>>(d, iters, mode, ratio, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double sec = ms / 5.0 * 1e-3;
    const double warps = (double)blocks * threads / 32;
    const double fw = mode == 0 ? warps : (mode == 1 ? 0 : (mode == 2 ? warps / 2 : warps));
    const double mw = mode == 1 ? warps : (mode == 0 ? 0 : (mode == 2 ? warps / 2 : warps));
    const double f_fl = fw * 32 * 8 * 2.0 * iters * (mode == 3 ? ratio : 1);
    const double m_fl = mw * 4 * 8 * 8 * 4 * 2.0 * iters;
    printf("%s\"mode%d_r%d\": {\"dfma_tf\": %.2f, \"dmma_tf\": %.2f, \"sum_tf\": %.2f}", mode + ratio > 0 ? ", " : "",
           mode, ratio, f_fl / sec / 1e12, m_fl / sec / 1e12, (f_fl + m_fl) / sec / 1e12);
  };
  printf("{");
  run(0, 0);
  run(1, 0);
  run(2, 0);
  run(3, 1);
  run(3, 2);
  run(3, 4);
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
