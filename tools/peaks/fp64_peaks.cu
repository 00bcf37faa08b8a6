// Microbenchmarks for the roofline denominators that MEASURED_PEAKS.json lacks:
// FP64 DFMA pipe peak, FP64 DMMA (mma.sync m8n8k4 f64) peak, FP32 FFMA peak,
// shared-memory LDS.128 bandwidth.  Run on one B200: prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void ffma_loop(float* out, int iters, float a, float b) {
  float x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678f) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void lds_loop(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 v = buf[(idx + j * 32) & 2047];
      acc.x += v.x; acc.y -= v.y;
    }
    idx = (idx + 256) & 2047;
  }
  if (acc.x == 12345.678) out[0] = acc.x + acc.y;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* d; float* f;
  CK(cudaMalloc(&d, 64)); CK(cudaMalloc(&f, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5.0;
  };
  const int blocks = nsm * 4, threads = 256, iters = 20000;
  double t = timeit([&] { dfma_loop<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7); });
  double dfma_tf = 2.0 * 8 * iters * (double)blocks * threads / (t * 1e-3) / 1e12;
  t = timeit([&] { ffma_loop<8><<<blocks, threads>>>(f, iters * 4, 0.999999f, 1e-7f); });
  double ffma_tf = 2.0 * 8 * iters * 4 * (double)blocks * threads / (t * 1e-3) / 1e12;
  t = timeit([&] { dmma_loop<<<blocks, threads>>>(d, iters); });
  double dmma_tf = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32) / (t * 1e-3) / 1e12;
  t = timeit([&] { lds_loop<<<blocks, threads>>>(d, iters); });
  double lds_tbs = 16.0 * 8 * (double)iters * blocks * threads / (t * 1e-3) / 1e12;
  CK(cudaGetLastError());
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"fp64_dfma_tflops\": %.2f, \"fp64_dmma_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, "
         "\"smem_lds128_tbs\": %.2f, \"sms\": %d, \"clock_attr_mhz\": %d}\n",
         dfma_tf, dmma_tf, ffma_tf, lds_tbs, nsm, clk / 1000);
  return 0;
}
