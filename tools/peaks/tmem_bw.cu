// TMEM read bandwidth on B200 with tcgen05.ld.32x32b.x4 (16 B per lane per
// load), and whether it contends with shared-memory LDS.128.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void tld4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
}
__device__ __forceinline__ void twait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

template <bool USE_TMEM, bool USE_SMEM>
__global__ void __launch_bounds__(1024, 1) bw(double* out, int iters) {
  __shared__ uint32_t taddr_s;
  __shared__ double2 buf[2048];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  double dacc = 0;
  int idx = lane;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[8][4];
    if (USE_TMEM) {
#pragma unroll
      for (int j = 0; j < 8; ++j) tld4(base + ((it * 8 + j) * 4 & 511), r[j][0], r[j][1], r[j][2], r[j][3]);
    }
    if (USE_SMEM) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double2 v = buf[(idx + j * 32 + warp * 128) & 2047];
        dacc += v.x - v.y;
      }
      idx = (idx + 7) & 2047;
    }
    if (USE_TMEM) {
      twait();
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += r[j][0] ^ r[j][1] ^ r[j][2] ^ r[j][3];
    }
  }
  if (acc == 12345u || dacc == 1.2345) out[0] = acc + dacc;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s));
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](const char* name, auto k, double bytes_per_iter_per_warp) {
    k<<<nsm, 1024>>>(d, 100);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(err)); return; }
    cudaEventRecord(e0);
    k<<<nsm, 1024>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double clk = ms * 1e-3 * 1.965e9;
    printf("%-10s %.3f ms  %.1f B/clk/SM\n", name, ms, 32.0 * iters * bytes_per_iter_per_warp / clk);
  };
  run("tmem", bw<true, false>, 8 * 512.0);
  run("smem", bw<false, true>, 8 * 512.0);
  run("both", bw<true, true>, 16 * 512.0);
  return 0;
}
