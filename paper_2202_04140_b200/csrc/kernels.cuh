// sm_100a kernels of the evaluator.
//
//   K1  pool_*          atomic basis A_{s,k} = sum_j phi_k(particle_j)   (evaluator.py:61-90)
//   K2  k2_*            recursive DAG program, fused c . A reduction      (evaluator.py:93-110,141)
//   K3  k3_naive        naive product basis, fused c . A reduction        (evaluator.py:113-121)
//   --  k_eval_nodes    every DAG node, bit-exact (no FMA)                (evaluator.py:93-110)
//   --  k_reduce_sites  deterministic per-output site sum (energy total)
//
// Layout: a CTA owns a tile of 32 sites; lane = site.  The pooled seeds the
// program references are staged ONCE per tile into shared memory as
// [slot][32 sites] complex (16 B per lane, conflict-free LDS.128); every warp
// of the CTA then walks its own chunk of the DFS program, with the DAG
// record stream read warp-uniformly (one broadcast L1 transaction per
// record) and the parent value of each level held in registers.  Only one
// secondary seed is fetched from shared memory per product.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.h"

namespace acedag {
namespace dev {

template <typename T> struct V2;
template <> struct V2<double> { using t = double2; };
template <> struct V2<float> { using t = float2; };

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// CPython _Py_c_prod with separate roundings (bit-identical to the reference)
__device__ __forceinline__ double2 cmul_exact(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

struct OpR {
  double c;
  uint32_t sa, sb, nch;
};

// 16-byte uniform record load (every lane reads the same address)
__device__ __forceinline__ OpR load_op(const Op* p) {
  int4 raw = __ldg(reinterpret_cast<const int4*>(p));
  OpR r;
  r.c = __hiloint2double(raw.y, raw.x);
  r.sa = (uint32_t)raw.z & 0xFFFFu;
  r.sb = (uint32_t)raw.z >> 16;
  r.nch = (uint32_t)raw.w;
  return r;
}

template <typename T, bool HYB>
struct SeedTab {
  using V = typename V2<T>::t;
  const V* s;   // shared  [Us][32]
  const V* g;   // global  [U-Us][32] (per-CTA cache of the cold tail)
  uint32_t us;
  int lane;
  __device__ __forceinline__ V operator()(uint32_t slot) const {
    if (!HYB || slot < us) return s[slot * 32 + lane];
    return g[(slot - us) * 32 + lane];
  }
};

// ---------------------------------------------------------------- K2 (fast)
// real coefficients, Re(phi), one output: acc += c * Re(v)
template <int D, int NU, typename T, bool HYB>
__device__ __forceinline__ void k2_visit(const Op*& op, uint32_t nch, typename V2<T>::t pv,
                                        T& acc0, T& acc1, const SeedTab<T, HYB>& tab) {
  using V = typename V2<T>::t;
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    // leaves of the deepest order: only the real part of the product
    uint32_t j = 0;
    for (; j + 4 <= nch; j += 4) {
      OpR r0 = load_op(op), r1 = load_op(op + 1), r2 = load_op(op + 2), r3 = load_op(op + 3);
      V s0 = tab(r0.sa), s1 = tab(r1.sa), s2 = tab(r2.sa), s3 = tab(r3.sa);
      acc0 += (T)r0.c * (s0.x * pv.x - s0.y * pv.y);
      acc1 += (T)r1.c * (s1.x * pv.x - s1.y * pv.y);
      acc0 += (T)r2.c * (s2.x * pv.x - s2.y * pv.y);
      acc1 += (T)r3.c * (s3.x * pv.x - s3.y * pv.y);
      op += 4;
    }
    for (; j < nch; ++j) {
      OpR r = load_op(op++);
      V s = tab(r.sa);
      acc0 += (T)r.c * (s.x * pv.x - s.y * pv.y);
    }
  } else {
    for (uint32_t j = 0; j < nch; ++j) {
      OpR r = load_op(op++);
      V v = cmul(tab(r.sa), pv);
      acc1 += (T)r.c * v.x;
      if (r.nch) k2_visit<D + 1, NU, T, HYB>(op, r.nch, v, acc0, acc1, tab);
    }
  }
}

template <int NU, typename T, bool HYB>
__global__ void __launch_bounds__(1024, 1)
k2_fast(const typename V2<T>::t* __restrict__ A, int64_t S, int L,
        const uint16_t* __restrict__ slot_label, int U, int Us, const Op* __restrict__ ops,
        const int32_t* __restrict__ chunk, double* __restrict__ out,
        typename V2<T>::t* __restrict__ gcache) {
  using V = typename V2<T>::t;
  extern __shared__ __align__(16) unsigned char smem[];
  V* sA = reinterpret_cast<V*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)Us * 32 * sizeof(V));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  V* gA = HYB ? gcache + (size_t)blockIdx.x * (U - Us) * 32 : nullptr;
  SeedTab<T, HYB> tab{sA, gA, (uint32_t)Us, lane};
  const int64_t ntiles = (S + 31) / 32;
  const Op* cbeg = ops + chunk[warp];
  const Op* cend = ops + chunk[warp + 1];
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t site = tile * 32 + lane;
    const bool valid = site < S;
    const V* row = A + (valid ? site : 0) * (int64_t)L;
    for (int u = warp; u < U; u += W) {
      V v = valid ? row[slot_label[u]] : V{0, 0};
      if (!HYB || u < Us) sA[u * 32 + lane] = v;
      else gA[(u - Us) * 32 + lane] = v;
    }
    __syncthreads();
    double acc = 0.0;
    for (const Op* op = cbeg; op < cend;) {
      T acc0 = 0, acc1 = 0;
      OpR r = load_op(op++);
      V a = tab(r.sa);
      V v = (r.sb == kSingle) ? a : cmul(a, tab(r.sb));
      acc0 += (T)r.c * v.x;
      if (r.nch) k2_visit<3, NU, T, HYB>(op, r.nch, v, acc0, acc1, tab);
      acc += (double)acc0 + (double)acc1;
    }
    red[warp * 32 + lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
      for (int w = 0; w < W; ++w) s += red[w * 32 + lane];
      if (valid) out[site] = s;
    }
  }
}

// ------------------------------------------------------------- K2 (general)
// complex coefficients and/or complex output and/or several outputs: NC
// complex accumulators per lane; coefficient table [n_ops, n_out].
template <int NC>
struct AccC {
  double re[NC], im[NC];
};

template <int D, int NU, int NC, bool HYB>
__device__ __forceinline__ void k2g_visit(const Op*& op, const Op* base, uint32_t nch, double2 pv,
                                         AccC<NC>& acc, const SeedTab<double, HYB>& tab,
                                         const double* cre, const double* cim, int n_out, int o0,
                                         int nc) {
  if constexpr (D > NU) {
    return;
  } else {
    for (uint32_t j = 0; j < nch; ++j) {
      const int64_t idx = op - base;
      OpR r = load_op(op++);
      double2 v = cmul(tab(r.sa), pv);
#pragma unroll
      for (int q = 0; q < NC; ++q)
        if (q < nc) {
          double c_r = __ldg(cre + idx * n_out + o0 + q);
          double c_i = cim ? __ldg(cim + idx * n_out + o0 + q) : 0.0;
          acc.re[q] += c_r * v.x - c_i * v.y;
          acc.im[q] += c_r * v.y + c_i * v.x;
        }
      if (r.nch) k2g_visit<D + 1, NU, NC, HYB>(op, base, r.nch, v, acc, tab, cre, cim, n_out, o0, nc);
    }
  }
}

template <int NU, int NC, bool HYB>
__global__ void __launch_bounds__(1024, 1)
k2_general(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label,
           int U, int Us, const Op* __restrict__ ops, const int32_t* __restrict__ chunk,
           const double* __restrict__ cre, const double* __restrict__ cim, int n_out, int o0,
           int complex_out, void* __restrict__ out, double2* __restrict__ gcache) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* sA = reinterpret_cast<double2*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)Us * 32 * sizeof(double2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U - Us) * 32 : nullptr;
  SeedTab<double, HYB> tab{sA, gA, (uint32_t)Us, lane};
  const int nc = min(NC, n_out - o0);
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t site = tile * 32 + lane;
    const bool valid = site < S;
    const double2* row = A + (valid ? site : 0) * (int64_t)L;
    for (int u = warp; u < U; u += W) {
      double2 v = valid ? row[slot_label[u]] : make_double2(0, 0);
      if (!HYB || u < Us) sA[u * 32 + lane] = v;
      else gA[(u - Us) * 32 + lane] = v;
    }
    __syncthreads();
    AccC<NC> acc;
#pragma unroll
    for (int q = 0; q < NC; ++q) acc.re[q] = acc.im[q] = 0.0;
    for (const Op* op = ops + chunk[warp]; op < ops + chunk[warp + 1];) {
      const int64_t idx = op - ops;
      OpR r = load_op(op++);
      double2 a = tab(r.sa);
      double2 v = (r.sb == kSingle) ? a : cmul(a, tab(r.sb));
#pragma unroll
      for (int q = 0; q < NC; ++q)
        if (q < nc) {
          double c_r = __ldg(cre + idx * n_out + o0 + q);
          double c_i = cim ? __ldg(cim + idx * n_out + o0 + q) : 0.0;
          acc.re[q] += c_r * v.x - c_i * v.y;
          acc.im[q] += c_r * v.y + c_i * v.x;
        }
      if (r.nch) k2g_visit<3, NU, NC, HYB>(op, ops, r.nch, v, acc, tab, cre, cim, n_out, o0, nc);
    }
    // reduce over warps, one output at a time, fixed order
    for (int q = 0; q < nc; ++q) {
      red[warp * 32 + lane] = acc.re[q];
      red[(W + warp) * 32 + lane] = acc.im[q];
      __syncthreads();
      if (warp == 0) {
        double sr = 0.0, si = 0.0;
        for (int w = 0; w < W; ++w) {
          sr += red[w * 32 + lane];
          si += red[(W + w) * 32 + lane];
        }
        if (valid) {
          if (complex_out) reinterpret_cast<double2*>(out)[site * n_out + o0 + q] = make_double2(sr, si);
          else reinterpret_cast<double*>(out)[site * n_out + o0 + q] = sr;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- K3 naive
// left-to-right product per coefficient node (evaluator.py:113-121)
template <int NU, bool GENERAL, bool HYB>
__global__ void __launch_bounds__(1024, 1)
k3_naive(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label,
         int U, int Us, const int32_t* __restrict__ seg, const uint16_t* __restrict__ slots,
         const double* __restrict__ cre, const double* __restrict__ cim, int n_out, int o0,
         int complex_out, void* __restrict__ out, double2* __restrict__ gcache) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* sA = reinterpret_cast<double2*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)Us * 32 * sizeof(double2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U - Us) * 32 : nullptr;
  SeedTab<double, HYB> tab{sA, gA, (uint32_t)Us, lane};
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t site = tile * 32 + lane;
    const bool valid = site < S;
    const double2* row = A + (valid ? site : 0) * (int64_t)L;
    for (int u = warp; u < U; u += W) {
      double2 v = valid ? row[slot_label[u]] : make_double2(0, 0);
      if (!HYB || u < Us) sA[u * 32 + lane] = v;
      else gA[(u - Us) * 32 + lane] = v;
    }
    __syncthreads();
    double ar = 0.0, ai = 0.0;
#pragma unroll
    for (int o = 1; o <= NU; ++o) {
      const int32_t b = seg[o], e = seg[o + 1];
      const int32_t n = e - b;
      const int32_t lo = b + (int32_t)((int64_t)n * warp / W), hi = b + (int32_t)((int64_t)n * (warp + 1) / W);
      for (int32_t rcd = lo; rcd < hi; ++rcd) {
        int4 sl = __ldg(reinterpret_cast<const int4*>(slots + (int64_t)rcd * kMaxOrder));
        uint32_t s[8] = {(uint32_t)sl.x & 0xFFFFu, (uint32_t)sl.x >> 16, (uint32_t)sl.y & 0xFFFFu,
                         (uint32_t)sl.y >> 16,     (uint32_t)sl.z & 0xFFFFu, (uint32_t)sl.z >> 16,
                         (uint32_t)sl.w & 0xFFFFu, (uint32_t)sl.w >> 16};
        double2 v = tab(s[0]);
#pragma unroll
        for (int t = 1; t < o; ++t) {
          if (!GENERAL && t == o - 1) {
            double2 w = tab(s[t]);
            v.x = v.x * w.x - v.y * w.y;  // last factor: real part only
          } else {
            v = cmul(v, tab(s[t]));
          }
        }
        const double c_r = __ldg(cre + (int64_t)rcd * n_out + o0);
        if (GENERAL) {
          const double c_i = cim ? __ldg(cim + (int64_t)rcd * n_out + o0) : 0.0;
          ar += c_r * v.x - c_i * v.y;
          ai += c_r * v.y + c_i * v.x;
        } else {
          ar += c_r * v.x;
        }
      }
    }
    red[warp * 32 + lane] = ar;
    red[(W + warp) * 32 + lane] = ai;
    __syncthreads();
    if (warp == 0) {
      double sr = 0.0, si = 0.0;
      for (int w = 0; w < W; ++w) {
        sr += red[w * 32 + lane];
        si += red[(W + w) * 32 + lane];
      }
      if (valid) {
        if (complex_out) reinterpret_cast<double2*>(out)[site * n_out + o0] = make_double2(sr, si);
        else reinterpret_cast<double*>(out)[site * n_out + o0] = sr;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ exact nodes
__global__ void k_eval_nodes(const double2* __restrict__ A, int64_t S, int L, int64_t N,
                             const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                             double2* __restrict__ vals) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    double2* row = vals + s * N;
    const double2* arow = A + s * (int64_t)L;
    for (int k = 0; k < L; ++k) row[k] = arow[k];
    for (int64_t k = L; k < N; ++k) row[k] = cmul_exact(row[__ldg(pa + k)], row[__ldg(pb + k)]);
  }
}

// naive_eval rows, bit-exact (evaluator.py:113-121)
__global__ void k_naive_products(const double2* __restrict__ vals, const int32_t* __restrict__ lens,
                                 int64_t n, int width, double2* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int len = lens ? lens[r] : width;
    double2 v = make_double2(1.0, 0.0);
    for (int t = 0; t < len; ++t) v = cmul_exact(v, vals[r * width + t]);
    out[r] = v;
  }
}

// ------------------------------------------------------- site reduction
__global__ void k_reduce_sites(const double* __restrict__ phi, int64_t S, int n_out,
                               double* __restrict__ total) {
  __shared__ double buf[1024];
  const int o = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < S; i += blockDim.x) s += phi[i * n_out + o];
  buf[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) buf[threadIdx.x] += buf[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) total[o] += buf[0];
}

}  // namespace dev
}  // namespace acedag
