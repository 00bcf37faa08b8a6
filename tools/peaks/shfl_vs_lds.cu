// Does SHFL share the shared-memory pipe with LDS on B200?  Times an LDS.128
// stream alone, a SHFL stream alone, and both interleaved.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lds_only(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { double2 v = buf[(idx + j * 32 + (threadIdx.x >> 5) * 256) & 2047]; acc.x += v.x; acc.y += v.y; }
    idx = (idx + 7) & 31;
  }
  if (acc.x == 1.2345) out[0] = acc.y;
}

__global__ void shfl_only(double* out, int iters) {
  int a = threadIdx.x, b = threadIdx.x * 3, c = threadIdx.x * 5, d = threadIdx.x * 7;
  int s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s += __shfl_sync(0xffffffffu, a, (j + it) & 31);
      a ^= s;
      s += __shfl_sync(0xffffffffu, b, (j + 3) & 31);
      s += __shfl_sync(0xffffffffu, c, (j + 5) & 31);
      s += __shfl_sync(0xffffffffu, d, (j + 7) & 31);
    }
  }
  if (s == 12345) out[0] = s;
}

__global__ void both(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x & 31;
  int a = threadIdx.x, b = threadIdx.x * 3, c = threadIdx.x * 5, d = threadIdx.x * 7, s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double2 v = buf[(idx + j * 32 + (threadIdx.x >> 5) * 256) & 2047]; acc.x += v.x; acc.y += v.y;
      s += __shfl_sync(0xffffffffu, a, (j + it) & 31);
      a ^= s;
      s += __shfl_sync(0xffffffffu, b, (j + 3) & 31);
      s += __shfl_sync(0xffffffffu, c, (j + 5) & 31);
      s += __shfl_sync(0xffffffffu, d, (j + 7) & 31);
    }
    idx = (idx + 7) & 31;
  }
  if (acc.x == 1.2345 || s == 12345) out[0] = acc.y + s;
}

__global__ void lds_bcast128(double* out, int iters) {
  __shared__ int4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_int4(i, i, i, i);
  __syncthreads();
  int s = 0, idx = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { int4 v = buf[(idx + j * 8) & 1023]; s += v.x ^ v.w; idx = (idx + v.y) & 1023; }
  }
  if (s == 12345) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = nsm * 2, threads = 1024, iters = 4000;
  auto run = [&](const char* name, auto k, double per_iter_units) {
    for (int w = 0; w < 2; ++w) k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e0); k<<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warp_ops = (double)blocks * (threads / 32) * iters * per_iter_units;
    double clk = ms * 1e-3 * 1.965e9;
    printf("%-14s %.3f ms  %.3f warp-instr/clk/SM\n", name, ms, warp_ops / clk / nsm);
  };
  run("lds128", lds_only, 8);
  run("shfl", shfl_only, 32);
  run("both(8lds+32shfl)", both, 40);
  run("lds128_bcast", lds_bcast128, 8);
  return 0;
}
