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

// fp64 products with a fixed contraction (explicit FMAs), so every kernel
// geometry computes the same value for a site
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
// Re(s * p)
__device__ __forceinline__ double re_mul(double2 s, double2 p) { return __fma_rn(s.x, p.x, -__dmul_rn(s.y, p.y)); }
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
  uint32_t off, nch, skip;
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// streaming read that should not displace the program stream from L1
template <typename V>
__device__ __forceinline__ V ld_stream(const V* p) {
  V v;
  if constexpr (sizeof(V) == 16) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  }
  return v;
}

// 16-byte uniform record load (every lane reads the same address)
__device__ __forceinline__ OpR load_op(const Op* p) {
  int4 raw = __ldg(reinterpret_cast<const int4*>(p));
  OpR r;
  r.c = __hiloint2double(raw.y, raw.x);
  r.off = (uint32_t)raw.z;
  r.nch = (uint32_t)raw.w & 0xFFFFu;
  r.skip = (uint32_t)raw.w >> 16;
  return r;
}

// Seed rows addressed by the byte offset stored in the record (c128 layout:
// slot * 512).  f32 tables use half the stride.  With HYB the rows past the
// shared-memory budget live in a per-CTA global cache (L1/L2 resident).
// Dynamic shared memory of every kernel in this file; kernels address it
// with 32-bit byte offsets so the loads compile to LDS [R + UR].
extern __shared__ __align__(16) unsigned char g_smem[];

template <typename T, bool HYB>
struct Seeds {
  using V = typename V2<T>::t;
  static constexpr int kShift = sizeof(V) == 16 ? 0 : 1;
  uint32_t s;      // g_smem byte offset of this lane's entry in row 0
  const char* g;   // global cache base + lane * sizeof(V) - us_bytes
  uint32_t us_bytes;
  __device__ __forceinline__ V operator()(uint32_t off) const {
    const uint32_t o = off >> kShift;
    if (!HYB || o < us_bytes) return *reinterpret_cast<const V*>(g_smem + s + o);
    return *reinterpret_cast<const V*>(g + o);
  }
};

// slot-indexed view used by the naive kernel
template <bool HYB>
struct SlotTab {
  const double2* s;
  const double2* g;
  uint32_t us;
  int lane;
  __device__ __forceinline__ double2 operator()(uint32_t slot) const {
    if (!HYB || slot < us) return s[slot * 32 + lane];
    return g[(slot - us) * 32 + lane];
  }
};

// Stage the seeds one tile references: lane = site, rows [slot][32 sites],
// plus the constant ONE row at slot U.  Rows past Us go to the global cache.
template <typename V, bool HYB>
__device__ __forceinline__ void stage_seeds(const V* __restrict__ A, int64_t S, int L, int64_t tile,
                                            const uint16_t* __restrict__ slot_label, int U, int Us,
                                            V* sA, V* gA, int warp, int W, int lane) {
  const int64_t site = tile * 32 + lane;
  const bool valid = site < S;
  const V* row = A + (valid ? site : 0) * (int64_t)L;
  for (int u = warp; u <= U; u += W) {
    V v;
    if (u == U) { v.x = 1; v.y = 0; }
    else if (valid) v = ld_stream(row + __ldg(slot_label + u));
    else { v.x = 0; v.y = 0; }
    if (!HYB || u < Us) sA[u * 32 + lane] = v;
    else gA[(u - Us) * 32 + lane] = v;
  }
}

// ---------------------------------------------------------------- K2 (fast)
// real coefficients, Re(phi), one output: acc += c * Re(v).
//
// Program stream: each warp walks a chunk of 16-byte records.  They are
// staged global -> registers -> a per-warp two-block shared ring (2 x 32
// records): one coalesced 512 B load per block, issued a block ahead, so the
// DFS never waits on L2; records are then read with broadcast LDS.128.
struct Stream {
  const int4* g;  // chunk start
  uint32_t ring;  // g_smem byte offset of this warp's ring [64 records]
  int4 stage;     // block b+2, one record per lane
  uint32_t i, n;  // next record, chunk length
  int lane;

  __device__ __forceinline__ int4 fetch(uint32_t q) const {
    return q < n ? __ldg(g + q) : make_int4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void put(uint32_t slot, int4 v) const {
    *reinterpret_cast<int4*>(g_smem + ring + (slot << 4)) = v;
  }
  __device__ __forceinline__ void begin(const int4* gp, uint32_t len, uint32_t r, int ln) {
    g = gp;
    n = len;
    ring = r;
    lane = ln;
    i = 0;
    const int4 b0 = fetch(lane), b1 = fetch(32 + lane);
    stage = fetch(64 + lane);
    __syncwarp();
    put(lane, b0);
    put(32 + lane, b1);
    __syncwarp();
  }
  __device__ __forceinline__ int4 at(uint32_t j) const {
    return *reinterpret_cast<const int4*>(g_smem + ring + (((i + j) & 63u) << 4));
  }
  __device__ __forceinline__ void advance(uint32_t k) {  // k <= 32
    const uint32_t ni = i + k;
    if ((ni >> 5) != (i >> 5)) {
      const uint32_t b = ni >> 5;
      __syncwarp();
      put(((b + 1) & 1) * 32 + lane, stage);
      stage = fetch((b + 2) * 32 + lane);
      __syncwarp();
    }
    i = ni;
  }
};

__device__ __forceinline__ double rec_c(int4 r) { return __hiloint2double(r.y, r.x); }
__device__ __forceinline__ uint32_t rec_off(int4 r) { return (uint32_t)r.z; }
__device__ __forceinline__ uint32_t rec_nch(int4 r) { return (uint32_t)r.w & 0xFFFFu; }

// Deepest level: the leaves of one parent as one batch (all record and seed
// loads in flight together); only the real part of each product is formed.
template <int K, typename T, bool HYB>
__device__ __forceinline__ void leaf_block(const Stream& st, typename V2<T>::t pv, T& acc0, T& acc1,
                                           const Seeds<T, HYB>& sd) {
  using V = typename V2<T>::t;
  int4 r[K];
  V s[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
#pragma unroll
  for (int j = 0; j < K; ++j) s[j] = sd(rec_off(r[j]));
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const T t = s[j].x * pv.x - s[j].y * pv.y;
    if (j & 1) acc1 += (T)rec_c(r[j]) * t;
    else acc0 += (T)rec_c(r[j]) * t;
  }
}

template <int MAXU, typename T, bool HYB>
__device__ __forceinline__ void leaves(Stream& st, uint32_t n, typename V2<T>::t pv, T& acc0, T& acc1,
                                       const Seeds<T, HYB>& sd) {
  while (n >= MAXU) {
    leaf_block<MAXU, T, HYB>(st, pv, acc0, acc1, sd);
    st.advance(MAXU);
    n -= MAXU;
  }
  switch (n) {
    case 1: leaf_block<1, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 2: leaf_block<2, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 3: leaf_block<3, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 4: if constexpr (MAXU > 4) leaf_block<4, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 5: if constexpr (MAXU > 5) leaf_block<5, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 6: if constexpr (MAXU > 6) leaf_block<6, T, HYB>(st, pv, acc0, acc1, sd); break;
    case 7: if constexpr (MAXU > 7) leaf_block<7, T, HYB>(st, pv, acc0, acc1, sd); break;
    default: break;
  }
  st.advance(n);
}

// Children of a node of order D-1 (values of order D), DFS preorder.
template <int D, int NU, int MAXU, typename T, bool HYB>
__device__ __forceinline__ void k2_visit(Stream& st, uint32_t n, typename V2<T>::t pv, T& acc0, T& acc1,
                                         const Seeds<T, HYB>& sd) {
  using V = typename V2<T>::t;
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves<MAXU, T, HYB>(st, n, pv, acc0, acc1, sd);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1);
      const V v = cmul(sd(rec_off(r)), pv);
      acc1 += (T)rec_c(r) * v.x;
      k2_visit<D + 1, NU, MAXU, T, HYB>(st, rec_nch(r), v, acc0, acc1, sd);
    }
  }
}

template <int NU, typename T, int WARPS, int MAXU, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_fast(const typename V2<T>::t* __restrict__ A, int64_t S, int L,
        const uint16_t* __restrict__ slot_label, int U, int Us, const Op* __restrict__ ops,
        const int32_t* __restrict__ chunk, int nchunk, double* __restrict__ out,
        typename V2<T>::t* __restrict__ gcache, double* __restrict__ part, int sched) {
  using V = typename V2<T>::t;
  unsigned char* smem = g_smem;
  V* sA = reinterpret_cast<V*>(smem);
  const uint32_t rings = (uint32_t)((size_t)Us * 32 * sizeof(V));
  int* next = reinterpret_cast<int*>(smem + rings + WARPS * 64 * 16);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  V* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 32 : nullptr;
  Seeds<T, HYB> sd;
  sd.s = (uint32_t)(lane * sizeof(V));
  sd.g = HYB ? reinterpret_cast<const char*>(gA) + lane * sizeof(V) - (size_t)Us * 32 * sizeof(V) : nullptr;
  sd.us_bytes = (uint32_t)((size_t)Us * 32 * sizeof(V));
  double* mypart = part + (size_t)blockIdx.x * nchunk * 32;
  const int4* prog = reinterpret_cast<const int4*>(ops);
  Stream st;
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    stage_seeds<V, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, WARPS, lane);
    if (threadIdx.x == 0) *next = 0;
    __syncthreads();
    // Chunk schedule.  sched == 0: static round robin (chunk c -> warp c % W),
    // one partial per warp.  sched == 1: dynamic (atomic counter), one
    // partial per chunk.  Both sum partials in a fixed order, so phi is
    // bitwise reproducible run to run.
    double wacc = 0.0;
    for (int k = 0;; ++k) {
      int ci;
      if (sched) {
        ci = 0;
        if (lane == 0) ci = atomicAdd(next, 1);
        ci = __shfl_sync(0xffffffffu, ci, 0);
      } else {
        ci = warp + k * WARPS;
      }
      if (ci >= nchunk) break;
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(prog + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      double acc = 0.0;
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        T acc0 = 0, acc1 = 0;
        const V v = cmul(sd(rec_off(r0)), sd(rec_off(r1)));
        acc0 += (T)rec_c(r0) * v.x;
        k2_visit<3, NU, MAXU, T, HYB>(st, rec_nch(r0), v, acc0, acc1, sd);
        acc += (double)acc0 + (double)acc1;
      }
      if (sched) mypart[ci * 32 + lane] = acc;
      else wacc += acc;
    }
    if (!sched) mypart[warp * 32 + lane] = wacc;
    __syncthreads();
    if (warp == 0) {
      const int np = sched ? nchunk : WARPS;
      double s = 0.0;
      for (int c = 0; c < np; ++c) s += __ldcg(mypart + c * 32 + lane);
      const int64_t site = tile * 32 + lane;
      if (site < S) out[site] = s;
    }
  }
}

// ------------------------------------------------ K2 (TMEM-resident seeds)
// The hot seed rows live in TENSOR MEMORY: TMEM reads (tcgen05.ld, 220 B/clk/
// SM measured) run on a path separate from the shared-memory crossbar
// (127 B/clk/SM), so the seed fetches no longer compete with the program
// stream.  TMEM is 128 lanes x 512 columns x 32 bit; a warp can only reach
// the 32 lanes of its quadrant (warp % 4), so the hot rows are replicated in
// all four quadrants: lane i of a quadrant = site i of the 32-site tile, a
// seed row = 4 columns (one complex128), 128 rows.  Slots >= kTmemRows (the
// cold tail, ~6% of fetches at cfg2) stay in shared memory / the global cache.
__device__ __forceinline__ void tmem_ld4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void tmem_st4(uint32_t addr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)),
               "r"(__double2hiint(v.y)));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ double2 u4_to_c(const uint32_t (&r)[4]) {
  return make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
}

template <bool HYB>
struct SeedsT {
  uint32_t tq;        // TMEM address of this warp's quadrant, column 0
  uint32_t s;         // g_smem byte offset of this lane's entry in cold row 0
  const char* g;      // global cache (rows past the smem budget)
  uint32_t us_rows;   // cold rows held in shared memory
  // records carry slot * 512; hot slots (< kTmemRows) are TMEM rows of 4 columns
  __device__ __forceinline__ void hot_issue(uint32_t off, uint32_t (&t)[4]) const {
    tmem_ld4(tq + (off >> 7), t);
  }
  __device__ __forceinline__ double2 hot(uint32_t off) const {
    uint32_t t[4];
    hot_issue(off, t);
    tmem_wait_ld();
    return u4_to_c(t);
  }
  __device__ __forceinline__ double2 cold(uint32_t off) const {
    const uint32_t c = off - kTmemRows * kRowBytes;  // byte offset of the cold row
    if (!HYB || c < us_rows * kRowBytes) return *reinterpret_cast<const double2*>(g_smem + s + c);
    return *reinterpret_cast<const double2*>(g + (c - us_rows * kRowBytes));
  }
  __device__ __forceinline__ double2 get(uint32_t off, bool is_hot) const { return is_hot ? hot(off) : cold(off); }
};

// one batch of K leaves whose seeds are all TMEM-resident
template <int K, bool HYB>
__device__ __forceinline__ void leaf_block_hot(const Stream& st, double2 pv, double& acc0, double& acc1,
                                               const SeedsT<HYB>& sd) {
  int4 r[K];
  uint32_t t[K][4];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
#pragma unroll
  for (int j = 0; j < K; ++j) sd.hot_issue((uint32_t)r[j].z, t[j]);
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double2 sv = u4_to_c(t[j]);
    const double tt = sv.x * pv.x - sv.y * pv.y;
    if (j & 1) acc1 += rec_c(r[j]) * tt;
    else acc0 += rec_c(r[j]) * tt;
  }
}

// one batch of K leaves whose seeds are in shared memory / the global cache
template <int K, bool HYB>
__device__ __forceinline__ void leaf_block_cold(const Stream& st, double2 pv, double& acc0, double& acc1,
                                                const SeedsT<HYB>& sd) {
  int4 r[K];
  double2 sv[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
#pragma unroll
  for (int j = 0; j < K; ++j) sv[j] = sd.cold((uint32_t)r[j].z);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double tt = sv[j].x * pv.x - sv[j].y * pv.y;
    if (j & 1) acc1 += rec_c(r[j]) * tt;
    else acc0 += rec_c(r[j]) * tt;
  }
}

template <bool HOT, int MAXU, bool HYB>
__device__ __forceinline__ void leaves_t(Stream& st, uint32_t n, double2 pv, double& acc0, double& acc1,
                                         const SeedsT<HYB>& sd) {
  while (n >= MAXU) {
    if constexpr (HOT) leaf_block_hot<MAXU, HYB>(st, pv, acc0, acc1, sd);
    else leaf_block_cold<MAXU, HYB>(st, pv, acc0, acc1, sd);
    st.advance(MAXU);
    n -= MAXU;
  }
  if (n) {
    if constexpr (MAXU > 2) {
      if (n >= 2) {
        if constexpr (HOT) leaf_block_hot<2, HYB>(st, pv, acc0, acc1, sd);
        else leaf_block_cold<2, HYB>(st, pv, acc0, acc1, sd);
        st.advance(2);
        n -= 2;
      }
    }
    if (n) {
      if constexpr (HOT) leaf_block_hot<1, HYB>(st, pv, acc0, acc1, sd);
      else leaf_block_cold<1, HYB>(st, pv, acc0, acc1, sd);
      st.advance(1);
    }
  }
}

// children of a node: n records, the first nh with TMEM-resident seeds
template <int D, int NU, int MAXU, bool HYB>
__device__ __forceinline__ void k2t_visit(Stream& st, uint32_t n, uint32_t nh, double2 pv, double& acc0,
                                          double& acc1, const SeedsT<HYB>& sd) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves_t<true, MAXU, HYB>(st, nh, pv, acc0, acc1, sd);
    leaves_t<false, MAXU, HYB>(st, n - nh, pv, acc0, acc1, sd);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1);
      const double2 v = cmul(sd.get((uint32_t)r.z, j < nh), pv);
      acc1 += rec_c(r) * v.x;
      k2t_visit<D + 1, NU, MAXU, HYB>(st, rec_nch(r), (uint32_t)r.w >> 16, v, acc0, acc1, sd);
    }
  }
}

// Records carry slot * 512 in .z (the generic program stream).
template <int NU, int WARPS, int MAXU, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_tmem(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
        int Us_cold, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
        double* __restrict__ out, double2* __restrict__ gcache, double* __restrict__ part) {
  unsigned char* smem = g_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;                                    // U seeds + ONE
  const int hot = rows < (int)kTmemRows ? rows : (int)kTmemRows;
  const int cold = rows - hot;
  const int us = cold < Us_cold ? cold : Us_cold;           // cold rows in smem
  double2* sC = reinterpret_cast<double2*>(smem);            // [us][32]
  const uint32_t rings = (uint32_t)((size_t)us * 512);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + rings + WARPS * 64 * 16);
  double2* gC = HYB ? gcache + (size_t)blockIdx.x * (cold - us) * 32 : nullptr;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  SeedsT<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gC) + lane * 16 : nullptr;
  sd.us_rows = (uint32_t)us;
  double* mypart = part + (size_t)blockIdx.x * WARPS * 32;
  Stream st;
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t site = tile * 32 + lane;
    const bool valid = site < S;
    const double2* row = A + (valid ? site : 0) * (int64_t)L;
    // hot rows -> TMEM, replicated per quadrant: warp w fills rows w/4, w/4 + W/4, ...
    for (int h = warp >> 2; h < hot; h += WARPS / 4) {
      double2 v;
      if (h == U) v = make_double2(1.0, 0.0);
      else v = valid ? ld_stream(row + __ldg(slot_label + h)) : make_double2(0.0, 0.0);
      tmem_st4(sd.tq + (uint32_t)h * 4, v);
    }
    // cold rows -> shared memory / global cache
    for (int c = warp; c < cold; c += WARPS) {
      const int u = hot + c;
      double2 v;
      if (u == U) v = make_double2(1.0, 0.0);
      else v = valid ? ld_stream(row + __ldg(slot_label + u)) : make_double2(0.0, 0.0);
      if (!HYB || c < us) sC[c * 32 + lane] = v;
      else gC[(size_t)(c - us) * 32 + lane] = v;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    double wacc = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        double acc0 = 0, acc1 = 0;
        const uint32_t fl = (uint32_t)r1.w >> 16;  // hot flags of the two root seeds
        const double2 v = cmul(sd.get((uint32_t)r0.z, fl & 1u), sd.get((uint32_t)r1.z, (fl >> 1) & 1u));
        acc0 += rec_c(r0) * v.x;
        k2t_visit<3, NU, MAXU, HYB>(st, rec_nch(r0), (uint32_t)r0.w >> 16, v, acc0, acc1, sd);
        wacc += acc0 + acc1;
      }
    }
    mypart[warp * 32 + lane] = wacc;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + w * 32 + lane);
      if (valid) out[site] = s;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// --------------------------------------- K2 (TMEM seeds, two sites per lane)
// 64-site tiles: lane holds sites t*64 + lane and t*64 + 32 + lane.  A hot
// TMEM row (64 rows, replicated per quadrant) is 8 columns = the seed of both
// sites, so ONE tcgen05.ld.32x32b.x8 serves two products.  Slots >= 64 come
// from shared memory rows [64 sites] (1 KB) or the global cache.
constexpr uint32_t kTmemRows2 = 64;

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
}
__device__ __forceinline__ void tmem_st8(uint32_t addr, double2 a, double2 b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(addr),
               "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)), "r"(__double2hiint(a.y)),
               "r"(__double2loint(b.x)), "r"(__double2hiint(b.x)), "r"(__double2loint(b.y)), "r"(__double2hiint(b.y)));
}

template <bool HYB>
struct SeedsT2 {
  uint32_t tq;        // TMEM address of this warp's quadrant, column 0
  uint32_t s;         // g_smem byte offset of this lane's entry (site A) in cold row 0
  const char* g;      // global cache base + lane * 16
  uint32_t us_rows;   // cold rows in shared memory
  __device__ __forceinline__ void hot_issue(uint32_t off, uint32_t (&t)[8]) const { tmem_ld8(tq + (off >> 6), t); }
  __device__ __forceinline__ void cold(uint32_t off, double2& a, double2& b) const {
    const uint32_t c = (off - kTmemRows2 * kRowBytes) * 2;  // byte offset of the 1 KB cold row
    if (!HYB || c < us_rows * 1024u) {
      a = *reinterpret_cast<const double2*>(g_smem + s + c);
      b = *reinterpret_cast<const double2*>(g_smem + s + c + 512);
    } else {
      a = *reinterpret_cast<const double2*>(g + (c - us_rows * 1024u));
      b = *reinterpret_cast<const double2*>(g + (c - us_rows * 1024u) + 512);
    }
  }
  __device__ __forceinline__ void get(uint32_t off, bool hot, double2& a, double2& b) const {
    if (hot) {
      uint32_t t[8];
      hot_issue(off, t);
      tmem_wait_ld();
      a = make_double2(__hiloint2double(t[1], t[0]), __hiloint2double(t[3], t[2]));
      b = make_double2(__hiloint2double(t[5], t[4]), __hiloint2double(t[7], t[6]));
    } else {
      cold(off, a, b);
    }
  }
};

template <bool HOT, int K, bool HYB>
__device__ __forceinline__ void leaf_block_t2(const Stream& st, double2 pa, double2 pb, double& acc0, double& acc1,
                                              const SeedsT2<HYB>& sd) {
  int4 r[K];
  double2 sa[K], sb[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
  if constexpr (HOT) {
    uint32_t t[K][8];
#pragma unroll
    for (int j = 0; j < K; ++j) sd.hot_issue((uint32_t)r[j].z, t[j]);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < K; ++j) {
      sa[j] = make_double2(__hiloint2double(t[j][1], t[j][0]), __hiloint2double(t[j][3], t[j][2]));
      sb[j] = make_double2(__hiloint2double(t[j][5], t[j][4]), __hiloint2double(t[j][7], t[j][6]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) sd.cold((uint32_t)r[j].z, sa[j], sb[j]);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double c = rec_c(r[j]);
    acc0 += c * (sa[j].x * pa.x - sa[j].y * pa.y);
    acc1 += c * (sb[j].x * pb.x - sb[j].y * pb.y);
  }
}

template <bool HOT, int MAXU, bool HYB>
__device__ __forceinline__ void leaves_t2(Stream& st, uint32_t n, double2 pa, double2 pb, double& acc0,
                                          double& acc1, const SeedsT2<HYB>& sd) {
  while (n >= MAXU) {
    leaf_block_t2<HOT, MAXU, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(MAXU);
    n -= MAXU;
  }
  if constexpr (MAXU > 2) {
    if (n >= 2) {
      leaf_block_t2<HOT, 2, HYB>(st, pa, pb, acc0, acc1, sd);
      st.advance(2);
      n -= 2;
    }
  }
  if (n) {
    leaf_block_t2<HOT, 1, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(1);
  }
}

template <int D, int NU, int MAXU, bool HYB>
__device__ __forceinline__ void k2t2_visit(Stream& st, uint32_t n, uint32_t nh, double2 pa, double2 pb,
                                           double& acc0, double& acc1, const SeedsT2<HYB>& sd) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves_t2<true, MAXU, HYB>(st, nh, pa, pb, acc0, acc1, sd);
    leaves_t2<false, MAXU, HYB>(st, n - nh, pa, pb, acc0, acc1, sd);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1);
      double2 sa, sb;
      sd.get((uint32_t)r.z, j < nh, sa, sb);
      const double2 va = cmul(sa, pa), vb = cmul(sb, pb);
      const double c = rec_c(r);
      acc0 += c * va.x;
      acc1 += c * vb.x;
      k2t2_visit<D + 1, NU, MAXU, HYB>(st, rec_nch(r), (uint32_t)r.w >> 16, va, vb, acc0, acc1, sd);
    }
  }
}

template <int NU, int WARPS, int MAXU, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_tmem2(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
         int Us_cold, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
         double* __restrict__ out, double2* __restrict__ gcache, double* __restrict__ part) {
  unsigned char* smem = g_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;
  const int hot = rows < (int)kTmemRows2 ? rows : (int)kTmemRows2;
  const int cold = rows - hot;
  const int us = cold < Us_cold ? cold : Us_cold;
  double2* sC = reinterpret_cast<double2*>(smem);            // [us][64]
  const uint32_t rings = (uint32_t)((size_t)us * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + rings + WARPS * 64 * 16);
  double2* gC = HYB ? gcache + (size_t)blockIdx.x * (cold - us) * 64 : nullptr;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  SeedsT2<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gC) + lane * 16 : nullptr;
  sd.us_rows = (uint32_t)us;
  double* mypart = part + (size_t)blockIdx.x * WARPS * 64;
  Stream st;
  const int64_t ntiles = (S + 63) / 64;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t sa_i = tile * 64 + lane, sb_i = sa_i + 32;
    const bool va_ok = sa_i < S, vb_ok = sb_i < S;
    const double2* rowa = A + (va_ok ? sa_i : 0) * (int64_t)L;
    const double2* rowb = A + (vb_ok ? sb_i : 0) * (int64_t)L;
    for (int h = warp >> 2; h < hot; h += WARPS / 4) {
      double2 a, b;
      if (h == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + h);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      tmem_st8(sd.tq + (uint32_t)h * 8, a, b);
    }
    for (int c = warp; c < cold; c += WARPS) {
      const int u = hot + c;
      double2 a, b;
      if (u == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + u);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      if (!HYB || c < us) {
        sC[c * 64 + lane] = a;
        sC[c * 64 + 32 + lane] = b;
      } else {
        gC[(size_t)(c - us) * 64 + lane] = a;
        gC[(size_t)(c - us) * 64 + 32 + lane] = b;
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    double wa = 0.0, wb = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        double acc0 = 0, acc1 = 0;
        const uint32_t fl = (uint32_t)r1.w >> 16;
        double2 a0, b0, a1, b1;
        sd.get((uint32_t)r0.z, fl & 1u, a0, b0);
        sd.get((uint32_t)r1.z, (fl >> 1) & 1u, a1, b1);
        const double2 va = cmul(a0, a1), vb = cmul(b0, b1);
        const double c = rec_c(r0);
        acc0 += c * va.x;
        acc1 += c * vb.x;
        k2t2_visit<3, NU, MAXU, HYB>(st, rec_nch(r0), (uint32_t)r0.w >> 16, va, vb, acc0, acc1, sd);
        wa += acc0;
        wb += acc1;
      }
    }
    mypart[(warp * 2 + 0) * 32 + lane] = wa;
    mypart[(warp * 2 + 1) * 32 + lane] = wb;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp < 2) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + (w * 2 + warp) * 32 + lane);
      const int64_t site = tile * 64 + warp * 32 + lane;
      if (site < S) out[site] = s;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// --------------------------- K2 (TMEM hot seeds, async program ring, v3)
// k2_tmem2 with a cheaper program stream: each warp's ring is three 32-record
// slots filled by cp.async one block ahead (no staging registers), records
// are addressed through a running shared-memory pointer with immediate
// offsets (two mirrored records after the last slot keep a two-record
// look-ahead contiguous), and block crossings are detected by a countdown.
struct Ring3 {
  static constexpr uint32_t kSlotBytes = 32 * 16, kBytes = 3 * kSlotBytes, kAlloc = kBytes + 2 * 16;
  const int4* g;     // next block to fetch
  const int4* gend;  // end of the chunk
  uint32_t p;        // shared address of the current record
  uint32_t base;     // shared address of slot 0
  int left;          // records left in the current block
  uint32_t nslot;    // slot the next fetched block goes to
  uint32_t i, n;     // records consumed, chunk length

  __device__ __forceinline__ void fetch(uint32_t slot, int lane) {
    const int4* src = g + lane;
    const bool ok = src < gend;
    const uint32_t sz = ok ? 16u : 0u;
    const int4* s = ok ? src : g;
    const uint32_t dst = base + slot * kSlotBytes + lane * 16;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(s), "r"(sz) : "memory");
    if (slot == 0 && lane < 2)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(base + kBytes + lane * 16), "l"(s),
                   "r"(sz)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    g += 32;
  }
  __device__ __forceinline__ void begin(const int4* gp, uint32_t len, uint32_t ring, int lane) {
    __syncwarp();  // the previous chunk's reads of this ring are done
    g = gp;
    gend = gp + len;
    base = ring;
    p = ring;
    left = 32;
    i = 0;
    n = len;
    fetch(0, lane);
    fetch(1, lane);
    fetch(2, lane);
    nslot = 0;
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
  }
  __device__ __forceinline__ int4 at(uint32_t j) const {
    int4 r;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(p + j * 16));
    return r;
  }
  __device__ __forceinline__ void advance(uint32_t k, int lane) {  // k <= 2
    p += k * 16;
    i += k;
    left -= (int)k;
    if (left <= 0) {
      left += 32;
      if (p >= base + kBytes) p -= kBytes;
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncwarp();
      fetch(nslot, lane);
      nslot = nslot == 2 ? 0 : nslot + 1;
    }
  }
};

template <bool HOT, int K, bool HYB>
__device__ __forceinline__ void leaf_block_t3(const Ring3& st, double2 pa, double2 pb, double& acc0, double& acc1,
                                              const SeedsT2<HYB>& sd) {
  int4 r[K];
  double2 sa[K], sb[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
  if constexpr (HOT) {
    uint32_t t[K][8];
#pragma unroll
    for (int j = 0; j < K; ++j) sd.hot_issue((uint32_t)r[j].z, t[j]);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < K; ++j) {
      sa[j] = make_double2(__hiloint2double(t[j][1], t[j][0]), __hiloint2double(t[j][3], t[j][2]));
      sb[j] = make_double2(__hiloint2double(t[j][5], t[j][4]), __hiloint2double(t[j][7], t[j][6]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) sd.cold((uint32_t)r[j].z, sa[j], sb[j]);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double c = rec_c(r[j]);
    acc0 = __fma_rn(c, re_mul(sa[j], pa), acc0);
    acc1 = __fma_rn(c, re_mul(sb[j], pb), acc1);
  }
}

template <bool HOT, bool HYB>
__device__ __forceinline__ void leaves_t3(Ring3& st, uint32_t n, double2 pa, double2 pb, double& acc0, double& acc1,
                                          const SeedsT2<HYB>& sd, int lane) {
  for (; n >= 2; n -= 2) {
    leaf_block_t3<HOT, 2, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(2, lane);
  }
  if (n) {
    leaf_block_t3<HOT, 1, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(1, lane);
  }
}

template <int D, int NU, bool HYB>
__device__ __forceinline__ void k2t3_visit(Ring3& st, uint32_t n, uint32_t nh, double2 pa, double2 pb,
                                           double& acc0, double& acc1, const SeedsT2<HYB>& sd, int lane) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves_t3<true, HYB>(st, nh, pa, pb, acc0, acc1, sd, lane);
    leaves_t3<false, HYB>(st, n - nh, pa, pb, acc0, acc1, sd, lane);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1, lane);
      double2 sa, sb;
      sd.get((uint32_t)r.z, j < nh, sa, sb);
      const double2 va = cmul(sa, pa), vb = cmul(sb, pb);
      const double c = rec_c(r);
      acc0 = __fma_rn(c, va.x, acc0);
      acc1 = __fma_rn(c, vb.x, acc1);
      k2t3_visit<D + 1, NU, HYB>(st, rec_nch(r), (uint32_t)r.w >> 16, va, vb, acc0, acc1, sd, lane);
    }
  }
}

// TILED: A is the tile-major table of k_tile_seeds<64> (as k2_quad)
template <int NU, int WARPS, bool HYB, bool TILED>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_tmem3(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
         int Us_cold, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
         double* __restrict__ out, double2* __restrict__ gcache, double* __restrict__ part, int64_t full_tiles,
         int tail_parts, double* __restrict__ tailbuf) {
  unsigned char* smem = g_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;
  const int hot = rows < (int)kTmemRows2 ? rows : (int)kTmemRows2;
  const int cold = rows - hot;
  const int us = cold < Us_cold ? cold : Us_cold;
  double2* sC = reinterpret_cast<double2*>(smem);  // [us][64]
  const uint32_t rings = (uint32_t)((size_t)us * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + rings + WARPS * Ring3::kAlloc);
  double2* gC = (HYB && !TILED) ? gcache + (size_t)blockIdx.x * (cold - us) * 64 : nullptr;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  SeedsT2<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gC) + lane * 16 : nullptr;
  sd.us_rows = (uint32_t)us;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem + rings + warp * Ring3::kAlloc);
  double* mypart = part + (size_t)blockIdx.x * nchunk * 64;
  Ring3 st;
  // whole tiles, then the last round's tiles split into program slices (k2_quad)
  const int64_t ntiles = (S + 63) / 64;
  const int64_t nitems = full_tiles + (ntiles - full_tiles) * tail_parts;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const bool whole = it < full_tiles;
    const int64_t tile = whole ? it : full_tiles + (it - full_tiles) / tail_parts;
    const int slice = whole ? 0 : (int)((it - full_tiles) % tail_parts);
    const int nsl = whole ? 1 : tail_parts;
    const int cb = (int)((int64_t)slice * nchunk / nsl), ce = (int)((int64_t)(slice + 1) * nchunk / nsl);
    const int64_t sa_i = tile * 64 + lane, sb_i = sa_i + 32;
    const bool va_ok = sa_i < S, vb_ok = sb_i < S;
    const double2* rowa = A + (va_ok ? sa_i : 0) * (int64_t)L;
    const double2* rowb = A + (vb_ok ? sb_i : 0) * (int64_t)L;
    if constexpr (TILED) {
      const double2* Tt = A + tile * (int64_t)rows * 64;
      if (HYB) sd.g = reinterpret_cast<const char*>(Tt + (size_t)(hot + us) * 64) + lane * 16;
      for (int h0 = warp >> 2; h0 < hot; h0 += 4 * (WARPS / 4)) {
        double2 v[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int h = h0 + q * (WARPS / 4);
#pragma unroll
          for (int k = 0; k < 2; ++k)
            v[q][k] = h < hot ? ld_stream(Tt + (size_t)h * 64 + k * 32 + lane) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int h = h0 + q * (WARPS / 4);
          if (h < hot) tmem_st8(sd.tq + (uint32_t)h * 8, v[q][0], v[q][1]);
        }
      }
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sC);
      for (int idx = threadIdx.x; idx < us * 64; idx += WARPS * 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + idx * 16),
                     "l"(Tt + (size_t)hot * 64 + idx)
                     : "memory");
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else {
    for (int h = warp >> 2; h < hot; h += WARPS / 4) {
      double2 a, b;
      if (h == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + h);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      tmem_st8(sd.tq + (uint32_t)h * 8, a, b);
    }
    for (int c = warp; c < cold; c += WARPS) {
      const int u = hot + c;
      double2 a, b;
      if (u == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + u);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      if (!HYB || c < us) {
        sC[c * 64 + lane] = a;
        sC[c * 64 + 32 + lane] = b;
      } else {
        gC[(size_t)(c - us) * 64 + lane] = a;
        gC[(size_t)(c - us) * 64 + 32 + lane] = b;
      }
    }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // one partial per (chunk, site), summed in chunk order: the result is
    // independent of the warp count, the tail split and the site count
    double* dst = whole ? mypart : tailbuf + (size_t)((it - full_tiles) / tail_parts) * nchunk * 64;
    for (int ci = cb + warp; ci < ce; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, (uint32_t)(e - b), ring, lane);
      double wa = 0.0, wb = 0.0;
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2, lane);
        const uint32_t fl = (uint32_t)r1.w >> 16;
        double2 a0, b0, a1, b1;
        sd.get((uint32_t)r0.z, fl & 1u, a0, b0);
        sd.get((uint32_t)r1.z, (fl >> 1) & 1u, a1, b1);
        const double2 va = cmul(a0, a1), vb = cmul(b0, b1);
        const double c = rec_c(r0);
        wa = __fma_rn(c, va.x, wa);
        wb = __fma_rn(c, vb.x, wb);
        k2t3_visit<3, NU, HYB>(st, rec_nch(r0), (uint32_t)r0.w >> 16, va, vb, wa, wb, sd, lane);
      }
      dst[(size_t)ci * 64 + lane] = wa;
      dst[(size_t)ci * 64 + 32 + lane] = wb;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (whole && threadIdx.x < 64) {
      double s = 0.0;
#pragma unroll 16
      for (int ci = 0; ci < nchunk; ++ci) s += __ldcg(mypart + (size_t)ci * 64 + threadIdx.x);
      const int64_t site = tile * 64 + threadIdx.x;
      if (site < S) out[site] = s;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// ------------------- K2 (TMEM hot seeds, three seed classes per node, v4)
// k2_tmem3 with the program re-encoded for this kernel (Op4): every node's
// children are ordered hot (TMEM) / shared-memory / global-cache by seed slot
// and the record carries the three counts, so each leaf run is three
// branch-free loops; seed locators are pre-scaled per class (TMEM column,
// shared byte offset, global byte offset); each chunk's root count bounds the
// root loop, so the ring keeps no record counter.
//   w (non-root and a root's first record): nch | nh << 11 | ns << 22
//   a root's second record w: class of seed a | class of seed b << 2
struct Ring4 {
  static constexpr uint32_t kSlotBytes = 32 * 16, kBytes = 3 * kSlotBytes, kAlloc = kBytes + 2 * 16;
  uint32_t p;   // shared address of the current record
  int left;     // records left in the current block
  uint32_t gi;  // next block to fetch (record index)
  uint32_t ge;  // end of the chunk (record index)

  __device__ __forceinline__ static void fetch(const int4* ops, uint32_t base, uint32_t slot, uint32_t gi,
                                               uint32_t ge, int lane) {
    const uint32_t q = gi + lane;
    const bool ok = q < ge;
    const int4* s = ops + (ok ? q : gi);
    const uint32_t sz = ok ? 16u : 0u;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(base + slot * kSlotBytes + lane * 16),
                 "l"(s), "r"(sz)
                 : "memory");
    if (slot == 0 && lane < 2)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(base + kBytes + lane * 16), "l"(s),
                   "r"(sz)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  __device__ __forceinline__ void begin(const int4* ops, uint32_t b, uint32_t e, uint32_t base, int lane) {
    __syncwarp();
    p = base;
    left = 32;
    ge = e;
    fetch(ops, base, 0, b, e, lane);
    fetch(ops, base, 1, b + 32, e, lane);
    fetch(ops, base, 2, b + 64, e, lane);
    gi = b + 96;
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
  }
  __device__ __forceinline__ int4 at(uint32_t j) const {
    int4 r;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(p + j * 16));
    return r;
  }
  // base: this warp's ring (recomputed by the caller only when crossing)
  template <typename BaseFn>
  __device__ __forceinline__ void advance(uint32_t k, const int4* ops, BaseFn base_fn, int lane) {
    p += k * 16;
    left -= (int)k;
    if (left <= 0) {
      left += 32;
      const uint32_t base = base_fn();
      if (p >= base + kBytes) p -= kBytes;
      // the slot just left is refilled with the block after the next one
      const uint32_t cur = (p - base) / kSlotBytes;
      const uint32_t freed = cur == 0 ? 2u : cur - 1;
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncwarp();
      fetch(ops, base, freed, gi, ge, lane);
      gi += 32;
    }
  }
};

template <bool HYB>
struct SeedsT4 {
  uint32_t tq;      // TMEM address of this warp's quadrant, column 0
  uint32_t sb;      // shared address of cold row 0, this lane's site A
  const char* gb;   // global cache of this tile, this lane's site A
  // class 0: TMEM column; 1: shared byte offset; 2: global byte offset
  __device__ __forceinline__ void hot_issue(uint32_t col, uint32_t (&t)[8]) const { tmem_ld8(tq + col, t); }
  __device__ __forceinline__ void smem(uint32_t off, double2& a, double2& b) const {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(a.x), "=d"(a.y) : "r"(sb + off));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(b.x), "=d"(b.y) : "r"(sb + off + 512));
  }
  __device__ __forceinline__ void glob(uint32_t off, double2& a, double2& b) const {
    a = *reinterpret_cast<const double2*>(gb + off);
    b = *reinterpret_cast<const double2*>(gb + off + 512);
  }
  __device__ __forceinline__ void get(uint32_t off, uint32_t cls, double2& a, double2& b) const {
    if (cls == 0) {
      uint32_t t[8];
      hot_issue(off, t);
      tmem_wait_ld();
      a = make_double2(__hiloint2double(t[1], t[0]), __hiloint2double(t[3], t[2]));
      b = make_double2(__hiloint2double(t[5], t[4]), __hiloint2double(t[7], t[6]));
    } else if (!HYB || cls == 1) {
      smem(off, a, b);
    } else {
      glob(off, a, b);
    }
  }
};

template <int CLS, int K, bool HYB>
__device__ __forceinline__ void leaf_block_t4(const Ring4& st, double2 pa, double2 pb, double& acc0, double& acc1,
                                              const SeedsT4<HYB>& sd) {
  int4 r[K];
  double2 sa[K], sb[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
  if constexpr (CLS == 0) {
    uint32_t t[K][8];
#pragma unroll
    for (int j = 0; j < K; ++j) sd.hot_issue((uint32_t)r[j].z, t[j]);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < K; ++j) {
      sa[j] = make_double2(__hiloint2double(t[j][1], t[j][0]), __hiloint2double(t[j][3], t[j][2]));
      sb[j] = make_double2(__hiloint2double(t[j][5], t[j][4]), __hiloint2double(t[j][7], t[j][6]));
    }
  } else if constexpr (CLS == 1) {
#pragma unroll
    for (int j = 0; j < K; ++j) sd.smem((uint32_t)r[j].z, sa[j], sb[j]);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) sd.glob((uint32_t)r[j].z, sa[j], sb[j]);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double c = rec_c(r[j]);
    acc0 += c * (sa[j].x * pa.x - sa[j].y * pa.y);
    acc1 += c * (sb[j].x * pb.x - sb[j].y * pb.y);
  }
}

template <int CLS, bool HYB, typename BaseFn>
__device__ __forceinline__ void leaves_t4(Ring4& st, uint32_t n, double2 pa, double2 pb, double& acc0,
                                          double& acc1, const SeedsT4<HYB>& sd, const int4* ops, BaseFn bf,
                                          int lane) {
  for (; n >= 2; n -= 2) {
    leaf_block_t4<CLS, 2, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(2, ops, bf, lane);
  }
  if (n) {
    leaf_block_t4<CLS, 1, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(1, ops, bf, lane);
  }
}

__device__ __forceinline__ uint32_t w4_nch(uint32_t w) { return w & 0x7FFu; }
__device__ __forceinline__ uint32_t w4_nh(uint32_t w) { return (w >> 11) & 0x7FFu; }
__device__ __forceinline__ uint32_t w4_ns(uint32_t w) { return w >> 22; }

template <int D, int NU, bool HYB, typename BaseFn>
__device__ __forceinline__ void k2t4_visit(Ring4& st, uint32_t w, double2 pa, double2 pb, double& acc0,
                                           double& acc1, const SeedsT4<HYB>& sd, const int4* ops, BaseFn bf,
                                           int lane) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    const uint32_t n = w4_nch(w), nh = w4_nh(w), ns = w4_ns(w);
    leaves_t4<0, HYB>(st, nh, pa, pb, acc0, acc1, sd, ops, bf, lane);
    leaves_t4<1, HYB>(st, ns, pa, pb, acc0, acc1, sd, ops, bf, lane);
    if (HYB) leaves_t4<2, HYB>(st, n - nh - ns, pa, pb, acc0, acc1, sd, ops, bf, lane);
  } else {
    const uint32_t n = w4_nch(w), nh = w4_nh(w), nhs = nh + w4_ns(w);
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1, ops, bf, lane);
      double2 sa, sb;
      sd.get((uint32_t)r.z, j < nh ? 0u : (j < nhs ? 1u : 2u), sa, sb);
      const double2 va = cmul(sa, pa), vb = cmul(sb, pb);
      const double c = rec_c(r);
      acc0 += c * va.x;
      acc1 += c * vb.x;
      k2t4_visit<D + 1, NU, HYB>(st, (uint32_t)r.w, va, vb, acc0, acc1, sd, ops, bf, lane);
    }
  }
}

template <int NU, int WARPS, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_tmem4(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
         int Us_cold, const Op* __restrict__ ops4, const int32_t* __restrict__ chunk,
         const int32_t* __restrict__ croots, int nchunk, double* __restrict__ out, double2* __restrict__ gcache,
         double* __restrict__ part) {
  unsigned char* smem = g_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;
  const int hot = rows < (int)kTmemRows2 ? rows : (int)kTmemRows2;
  const int cold = rows - hot;
  const int us = cold < Us_cold ? cold : Us_cold;
  double2* sC = reinterpret_cast<double2*>(smem);  // [us][64]
  const uint32_t rings = (uint32_t)((size_t)us * 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + rings + WARPS * Ring4::kAlloc);
  double2* gC = HYB ? gcache + (size_t)blockIdx.x * (cold - us) * 64 : nullptr;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  SeedsT4<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.sb = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(lane * 16);
  sd.gb = HYB ? reinterpret_cast<const char*>(gC) + lane * 16 : nullptr;
  const int4* ops = reinterpret_cast<const int4*>(ops4);
  auto ring_base = [=]() {
    return (uint32_t)__cvta_generic_to_shared(g_smem) + rings + (uint32_t)((threadIdx.x >> 5) * Ring4::kAlloc);
  };
  double* mypart = part + (size_t)blockIdx.x * WARPS * 64;
  Ring4 st;
  const int64_t ntiles = (S + 63) / 64;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t sa_i = tile * 64 + lane, sb_i = sa_i + 32;
    const bool va_ok = sa_i < S, vb_ok = sb_i < S;
    const double2* rowa = A + (va_ok ? sa_i : 0) * (int64_t)L;
    const double2* rowb = A + (vb_ok ? sb_i : 0) * (int64_t)L;
    for (int h = warp >> 2; h < hot; h += WARPS / 4) {
      double2 a, b;
      if (h == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + h);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      tmem_st8(sd.tq + (uint32_t)h * 8, a, b);
    }
    for (int c = warp; c < cold; c += WARPS) {
      const int u = hot + c;
      double2 a, b;
      if (u == U) {
        a = b = make_double2(1.0, 0.0);
      } else {
        const int lab = __ldg(slot_label + u);
        a = va_ok ? ld_stream(rowa + lab) : make_double2(0.0, 0.0);
        b = vb_ok ? ld_stream(rowb + lab) : make_double2(0.0, 0.0);
      }
      if (!HYB || c < us) {
        sC[c * 64 + lane] = a;
        sC[c * 64 + 32 + lane] = b;
      } else {
        gC[(size_t)(c - us) * 64 + lane] = a;
        gC[(size_t)(c - us) * 64 + 32 + lane] = b;
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    double wa = 0.0, wb = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      const int32_t nr = __ldg(croots + ci);
      st.begin(ops, (uint32_t)b, (uint32_t)e, ring_base(), lane);
      for (int32_t k = 0; k < nr; ++k) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2, ops, ring_base, lane);
        const uint32_t fl = (uint32_t)r1.w;
        double2 a0, b0, a1, b1;
        sd.get((uint32_t)r0.z, fl & 3u, a0, b0);
        sd.get((uint32_t)r1.z, (fl >> 2) & 3u, a1, b1);
        const double2 va = cmul(a0, a1), vb = cmul(b0, b1);
        const double c = rec_c(r0);
        wa += c * va.x;
        wb += c * vb.x;
        k2t4_visit<3, NU, HYB>(st, (uint32_t)r0.w, va, vb, wa, wb, sd, ops, ring_base, lane);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    mypart[(warp * 2 + 0) * 32 + lane] = wa;
    mypart[(warp * 2 + 1) * 32 + lane] = wb;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp < 2) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + (w * 2 + warp) * 32 + lane);
      const int64_t site = tile * 64 + warp * 32 + lane;
      if (site < S) out[site] = s;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// --------------------------------------------- tile-major seed table (K2 input)
// A [S, L] c128 -> T [ntiles][U + 1][TS] c128: row r of tile t holds slot r
// (row U = the constant ONE) for the TS sites of the tile, so the K2 kernels
// stage and fetch whole rows with coalesced loads.  Lanes walk the used
// columns in ascending order (coalesced reads of each site row); a padded
// [32][TS + 1] shared block transposes 32 columns at a time.
// cols: column of the j-th used entry (NULL: j); slots: its row (NULL: j).
template <int TS, typename V = double2>
__global__ void __launch_bounds__(512) k_tile_seeds(const V* __restrict__ A, int64_t S, int L,
                                                    const int32_t* __restrict__ cols,
                                                    const uint16_t* __restrict__ slots, int U,
                                                    V* __restrict__ T) {
  extern __shared__ __align__(16) unsigned char tbraw[];
  V* tb = reinterpret_cast<V*>(tbraw);  // [32][TS + 1]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = 16;
  const int64_t tile = blockIdx.x;
  const int R = U + 1;
  V* Tt = T + tile * (int64_t)R * TS;
  for (int j0 = 0; j0 < U; j0 += 32) {
    const int j = j0 + lane;
    const int col = j < U ? (cols ? __ldg(cols + j) : j) : -1;
    V v[TS / NW];
#pragma unroll
    for (int q = 0; q < TS / NW; ++q) {
      const int64_t site = tile * TS + warp + q * NW;
      v[q] = (col >= 0 && site < S) ? ld_stream(A + site * L + col) : V{0, 0};
    }
#pragma unroll
    for (int q = 0; q < TS / NW; ++q) tb[lane * (TS + 1) + warp + q * NW] = v[q];
    __syncthreads();
    for (int jj = warp; jj < 32 && j0 + jj < U; jj += NW) {
      const int slot = slots ? (int)__ldg(slots + j0 + jj) : j0 + jj;
#pragma unroll
      for (int q = 0; q < TS / 32; ++q) Tt[(int64_t)slot * TS + q * 32 + lane] = tb[jj * (TS + 1) + q * 32 + lane];
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < TS; q += blockDim.x) Tt[(int64_t)U * TS + q] = V{1, 0};
}

// ------------------------------------- K2 (four sites per lane, TMEM + smem)
// 128-site tiles: lane l handles sites l, l+32, l+64, l+96 of the tile, so
// every program record (its load, decode, seed addressing and loop control)
// serves four sites -- the per-record overhead that bounds k2_tmem2/3 is
// amortised twice as far.  Seed rows are 2 KB ([4][32] c128): the 32 hottest
// in TMEM (16 columns per lane, one x16 load per fetch, replicated per lane
// quadrant), the next in shared memory, the tail in the per-CTA global
// cache.  16 warps x 128 registers.
constexpr uint32_t kTmemRowsQ = 32;

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}

struct C4 {
  double2 v[4];
};

template <bool HYB>
struct SeedsQ {
  uint32_t tq;      // TMEM address of this warp's quadrant, column 0
  uint32_t sb;      // shared address of cold row 0 + lane * 16
  const char* gb;   // global cache of this CTA + lane * 16
  uint32_t usB;     // shared-memory cold rows * 2048
  // records carry slot * 512: hot slot s -> TMEM column 16 s; cold -> 2 KB row
  __device__ __forceinline__ void hot_issue(uint32_t off, uint32_t (&t)[16]) const { tmem_ld16(tq + (off >> 5), t); }
  __device__ __forceinline__ static C4 unpack(const uint32_t (&t)[16]) {
    C4 s;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      s.v[k] = make_double2(__hiloint2double(t[4 * k + 1], t[4 * k]), __hiloint2double(t[4 * k + 3], t[4 * k + 2]));
    return s;
  }
  __device__ __forceinline__ C4 cold(uint32_t off) const {
    const uint32_t c = off * 4 - kTmemRowsQ * 2048;  // byte offset of the 2 KB cold row
    C4 s;
    if (!HYB || c < usB) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(s.v[k].x), "=d"(s.v[k].y) : "r"(sb + c + k * 512));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) s.v[k] = *reinterpret_cast<const double2*>(gb + (c - usB) + k * 512);
    }
    return s;
  }
  __device__ __forceinline__ C4 get(uint32_t off, bool hot) const {
    if (hot) {
      uint32_t t[16];
      hot_issue(off, t);
      tmem_wait_ld();
      return unpack(t);
    }
    return cold(off);
  }
};

__device__ __forceinline__ C4 cmul4(const C4& a, const C4& b) {
  C4 r;
#pragma unroll
  for (int k = 0; k < 4; ++k) r.v[k] = cmul(a.v[k], b.v[k]);
  return r;
}

template <bool HOT, int K, bool HYB>
__device__ __forceinline__ void leaf_block_q(const Ring3& st, const C4& pv, double (&acc)[4], const SeedsQ<HYB>& sd) {
  int4 r[K];
  C4 s[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
  if constexpr (HOT) {
    uint32_t t[K][16];
#pragma unroll
    for (int j = 0; j < K; ++j) sd.hot_issue((uint32_t)r[j].z, t[j]);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = SeedsQ<HYB>::unpack(t[j]);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = sd.cold((uint32_t)r[j].z);
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double c = rec_c(r[j]);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = __fma_rn(c, re_mul(s[j].v[k], pv.v[k]), acc[k]);
  }
}

template <bool HOT, int MAXU, bool HYB>
__device__ __forceinline__ void leaves_q(Ring3& st, uint32_t n, const C4& pv, double (&acc)[4], const SeedsQ<HYB>& sd,
                                         int lane) {
  if constexpr (MAXU >= 2) {
    for (; n >= 2; n -= 2) {
      leaf_block_q<HOT, 2, HYB>(st, pv, acc, sd);
      st.advance(2, lane);
    }
  }
  for (; n; --n) {
    leaf_block_q<HOT, 1, HYB>(st, pv, acc, sd);
    st.advance(1, lane);
  }
}

template <int D, int NU, int MAXU, bool HYB>
__device__ __forceinline__ void k2q_visit(Ring3& st, uint32_t n, uint32_t nh, const C4& pv, double (&acc)[4],
                                          const SeedsQ<HYB>& sd, int lane) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves_q<true, MAXU, HYB>(st, nh, pv, acc, sd, lane);
    leaves_q<false, MAXU, HYB>(st, n - nh, pv, acc, sd, lane);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1, lane);
      const C4 v = cmul4(sd.get((uint32_t)r.z, j < nh), pv);
      const double c = rec_c(r);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = __fma_rn(c, v.v[k].x, acc[k]);
      k2q_visit<D + 1, NU, MAXU, HYB>(st, rec_nch(r), (uint32_t)r.w >> 16, v, acc, sd, lane);
    }
  }
}

// TILED: A is the tile-major table of k_tile_seeds (rows staged with
// coalesced loads; the global-cache tail is read from it in place)
template <int NU, int WARPS, int MAXU, bool HYB, bool TILED>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_quad(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
        int Us_cold, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
        double* __restrict__ out, double2* __restrict__ gcache, double* __restrict__ part, int64_t full_tiles,
        int tail_parts, double* __restrict__ tailbuf) {
  unsigned char* smem = g_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;
  const int hot = rows < (int)kTmemRowsQ ? rows : (int)kTmemRowsQ;
  const int cold = rows - hot;
  const int us = cold < Us_cold ? cold : Us_cold;
  double2* sC = reinterpret_cast<double2*>(smem);  // [us][128]
  const uint32_t rings = (uint32_t)((size_t)us * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + rings + WARPS * Ring3::kAlloc);
  int* dyn = reinterpret_cast<int*>(tslot) + 1;        // next chunk of the current item
  int32_t* slab = reinterpret_cast<int32_t*>(tslot) + 4;  // slot -> label (-1: the ONE row)
  for (int h = threadIdx.x; h < rows; h += blockDim.x) slab[h] = h == U ? -1 : (int32_t)__ldg(slot_label + h);
  double2* gC = (HYB && !TILED) ? gcache + (size_t)blockIdx.x * (cold - us) * 128 : nullptr;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  SeedsQ<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.sb = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(lane * 16);
  sd.gb = HYB ? reinterpret_cast<const char*>(gC) + lane * 16 : nullptr;
  sd.usB = (uint32_t)us * 2048u;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem + rings + warp * Ring3::kAlloc);
  double* mypart = part + (size_t)blockIdx.x * nchunk * 128;
  Ring3 st;
  // work items: whole tiles, then the last partial round's tiles split into
  // tail_parts program slices each (partial sums to tailbuf, summed in slice
  // order by k_tail_reduce) so the final round still fills the grid
  const int64_t ntiles = (S + 127) / 128;
  const int64_t nitems = full_tiles + (ntiles - full_tiles) * tail_parts;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const bool whole = it < full_tiles;
    const int64_t tile = whole ? it : full_tiles + (it - full_tiles) / tail_parts;
    const int slice = whole ? 0 : (int)((it - full_tiles) % tail_parts);
    const int nsl = whole ? 1 : tail_parts;
    const int cb = (int)((int64_t)slice * nchunk / nsl), ce = (int)((int64_t)(slice + 1) * nchunk / nsl);
    const double2* row[4];
    bool ok[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t s = tile * 128 + k * 32 + lane;
      ok[k] = s < S;
      row[k] = A + (ok[k] ? s : 0) * (int64_t)L;
    }
    const double2* Tt = A + tile * (int64_t)rows * 128;  // TILED: this tile's rows
    if (TILED && HYB) sd.gb = reinterpret_cast<const char*>(Tt + (size_t)(hot + us) * 128) + lane * 16;
    if constexpr (TILED) {
      for (int h0 = warp >> 2; h0 < hot; h0 += 4 * (WARPS / 4)) {
        double2 v[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int h = h0 + q * (WARPS / 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) v[q][k] = h < hot ? ld_stream(Tt + (size_t)h * 128 + k * 32 + lane) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int h = h0 + q * (WARPS / 4);
          if (h < hot) {
            tmem_st8(sd.tq + (uint32_t)h * 16, v[q][0], v[q][1]);
            tmem_st8(sd.tq + (uint32_t)h * 16 + 8, v[q][2], v[q][3]);
          }
        }
      }
      // shared-memory rows: asynchronous 16-byte copies, no registers
      const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sC);
      for (int idx = threadIdx.x; idx < us * 128; idx += WARPS * 32) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + idx * 16),
                     "l"(Tt + (size_t)hot * 128 + idx)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else {
    // staging: four rows per pass, sixteen loads in flight per lane
    for (int h0 = warp >> 2; h0 < hot; h0 += 4 * (WARPS / 4)) {
      double2 v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (WARPS / 4);
        const int lab = h < hot ? slab[h] : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[q][k] = (lab >= 0 && ok[k]) ? ld_stream(row[k] + lab) : make_double2(h == U ? 1.0 : 0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (WARPS / 4);
        if (h < hot) {
          tmem_st8(sd.tq + (uint32_t)h * 16, v[q][0], v[q][1]);
          tmem_st8(sd.tq + (uint32_t)h * 16 + 8, v[q][2], v[q][3]);
        }
      }
    }
    for (int c0 = warp; c0 < cold; c0 += 4 * WARPS) {
      double2 v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + q * WARPS;
        const int lab = c < cold ? slab[hot + c] : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[q][k] = (lab >= 0 && ok[k]) ? ld_stream(row[k] + lab) : make_double2(hot + c == U ? 1.0 : 0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + q * WARPS;
        if (c < cold) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (!HYB || c < us) sC[c * 128 + k * 32 + lane] = v[q][k];
            else gC[(size_t)(c - us) * 128 + k * 32 + lane] = v[q][k];
          }
        }
      }
    }
    }
    if (threadIdx.x == 0) *dyn = cb + WARPS;
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // one partial per (chunk, site), summed in chunk order (as k2_tmem3)
    double* dst = whole ? mypart : tailbuf + (size_t)((it - full_tiles) / tail_parts) * nchunk * 128;
    // chunks handed out dynamically (the partials are indexed by chunk, so
    // the result does not depend on which warp ran which chunk)
    for (int ci = cb + warp; ci < ce;) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, (uint32_t)(e - b), ring, lane);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2, lane);
        const uint32_t fl = (uint32_t)r1.w >> 16;
        const C4 v = cmul4(sd.get((uint32_t)r0.z, fl & 1u), sd.get((uint32_t)r1.z, (fl >> 1) & 1u));
        const double c = rec_c(r0);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fma_rn(c, v.v[k].x, acc[k]);
        k2q_visit<3, NU, MAXU, HYB>(st, rec_nch(r0), (uint32_t)r0.w >> 16, v, acc, sd, lane);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[(size_t)ci * 128 + k * 32 + lane] = acc[k];
      int nx = 0;
      if (lane == 0) nx = atomicAdd(dyn, 1);
      ci = __shfl_sync(0xffffffffu, nx, 0);
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (whole && threadIdx.x < 128) {
      double s = 0.0;
#pragma unroll 16
      for (int ci = 0; ci < nchunk; ++ci) s += __ldcg(mypart + (size_t)ci * 128 + threadIdx.x);
      const int64_t site = tile * 128 + threadIdx.x;
      if (site < S) out[site] = s;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// tail tiles: out[site] = sum over chunks (in chunk order) of the partials
__global__ void k_tail_reduce(const double* __restrict__ tailbuf, int64_t first_site, int64_t S, int tile_sites,
                              int nchunk, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // site offset past first_site
  if (first_site + i >= S) return;
  const int64_t t = i / tile_sites, o = i % tile_sites;
  const double* p = tailbuf + t * nchunk * tile_sites + o;
  double s = 0.0;
#pragma unroll 16
  for (int c = 0; c < nchunk; ++c) s += p[(size_t)c * tile_sites];
  out[first_site + i] = s;
}

// ------------------------------------------------------ K2 (two sites/lane)
// 64-site tiles: lane handles sites t*64 + lane and t*64 + 32 + lane, so each
// program record (and its decode) serves twice the sites.  The seed table is
// [slot][64 sites] c128 (1 KB rows); the hottest rows (98% of fetches at
// cfg2/cfg5) stay in shared memory, the cold tail in the per-CTA global cache.
template <typename T, bool HYB>
struct Seeds2 {
  using V = typename V2<T>::t;
  static constexpr uint32_t kRow = 64 * sizeof(V);  // bytes per slot row
  uint32_t s;         // g_smem byte offset of this lane's entry (first half) in row 0
  const char* g;      // global cache base + lane * sizeof(V) - us_bytes
  uint32_t us_bytes;  // smem rows * kRow
  __device__ __forceinline__ void operator()(uint32_t off, V& a, V& b) const {
    const uint32_t o = (off / kRowBytes) * kRow;  // records carry slot * 512
    if (!HYB || o < us_bytes) {
      a = *reinterpret_cast<const V*>(g_smem + s + o);
      b = *reinterpret_cast<const V*>(g_smem + s + o + 32 * sizeof(V));
    } else {
      a = *reinterpret_cast<const V*>(g + o);
      b = *reinterpret_cast<const V*>(g + o + 32 * sizeof(V));
    }
  }
};

template <int K, typename T, bool HYB>
__device__ __forceinline__ void leaf_block2(const Stream& st, typename V2<T>::t pa, typename V2<T>::t pb,
                                            T& acc0, T& acc1, const Seeds2<T, HYB>& sd) {
  using V = typename V2<T>::t;
  int4 r[K];
  V sa[K], sb[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
#pragma unroll
  for (int j = 0; j < K; ++j) sd(rec_off(r[j]), sa[j], sb[j]);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const T c = (T)rec_c(r[j]);
    acc0 += c * (sa[j].x * pa.x - sa[j].y * pa.y);
    acc1 += c * (sb[j].x * pb.x - sb[j].y * pb.y);
  }
}

template <int MAXU, typename T, bool HYB>
__device__ __forceinline__ void leaves2(Stream& st, uint32_t n, typename V2<T>::t pa, typename V2<T>::t pb,
                                        T& acc0, T& acc1, const Seeds2<T, HYB>& sd) {
  while (n >= MAXU) {
    leaf_block2<MAXU, T, HYB>(st, pa, pb, acc0, acc1, sd);
    st.advance(MAXU);
    n -= MAXU;
  }
  switch (n) {
    case 1: leaf_block2<1, T, HYB>(st, pa, pb, acc0, acc1, sd); break;
    case 2: if constexpr (MAXU > 2) leaf_block2<2, T, HYB>(st, pa, pb, acc0, acc1, sd); break;
    case 3: if constexpr (MAXU > 3) leaf_block2<3, T, HYB>(st, pa, pb, acc0, acc1, sd); break;
    default: break;
  }
  st.advance(n);
}

template <int D, int NU, int MAXU, typename T, bool HYB>
__device__ __forceinline__ void k2_visit2(Stream& st, uint32_t n, typename V2<T>::t pa, typename V2<T>::t pb,
                                          T& acc0, T& acc1, const Seeds2<T, HYB>& sd) {
  using V = typename V2<T>::t;
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    leaves2<MAXU, T, HYB>(st, n, pa, pb, acc0, acc1, sd);
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1);
      V sa, sb;
      sd(rec_off(r), sa, sb);
      const V va = cmul(sa, pa), vb = cmul(sb, pb);
      const T c = (T)rec_c(r);
      acc0 += c * va.x;
      acc1 += c * vb.x;
      k2_visit2<D + 1, NU, MAXU, T, HYB>(st, rec_nch(r), va, vb, acc0, acc1, sd);
    }
  }
}

// stage 64 sites: lane covers sites lane and 32 + lane of the tile
template <typename V, bool HYB>
__device__ __forceinline__ void stage_seeds2(const V* __restrict__ A, int64_t S, int L, int64_t tile,
                                             const uint16_t* __restrict__ slot_label, int U, int Us,
                                             V* sA, V* gA, int warp, int W, int lane) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t site = tile * 64 + h * 32 + lane;
    const bool valid = site < S;
    const V* row = A + (valid ? site : 0) * (int64_t)L;
    for (int u = warp; u <= U; u += W) {
      V v;
      if (u == U) { v.x = 1; v.y = 0; }
      else if (valid) v = ld_stream(row + __ldg(slot_label + u));
      else { v.x = 0; v.y = 0; }
      if (!HYB || u < Us) sA[u * 64 + h * 32 + lane] = v;
      else gA[(u - Us) * 64 + h * 32 + lane] = v;
    }
  }
}

template <int NU, typename T, int WARPS, int MAXU, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_fast2(const typename V2<T>::t* __restrict__ A, int64_t S, int L,
         const uint16_t* __restrict__ slot_label, int U, int Us, const Op* __restrict__ ops,
         const int32_t* __restrict__ chunk, int nchunk, double* __restrict__ out,
         typename V2<T>::t* __restrict__ gcache, double* __restrict__ part) {
  using V = typename V2<T>::t;
  unsigned char* smem = g_smem;
  V* sA = reinterpret_cast<V*>(smem);
  const uint32_t rings = (uint32_t)((size_t)Us * 64 * sizeof(V));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  V* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 64 : nullptr;
  Seeds2<T, HYB> sd;
  sd.s = (uint32_t)(lane * sizeof(V));
  sd.g = HYB ? reinterpret_cast<const char*>(gA) + lane * sizeof(V) - (size_t)Us * 64 * sizeof(V) : nullptr;
  sd.us_bytes = (uint32_t)((size_t)Us * 64 * sizeof(V));
  double* mypart = part + (size_t)blockIdx.x * WARPS * 64;
  Stream st;
  const int64_t ntiles = (S + 63) / 64;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    stage_seeds2<V, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, WARPS, lane);
    __syncthreads();
    double wa = 0.0, wb = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        T acc0 = 0, acc1 = 0;
        V a0, b0, a1, b1;
        sd(rec_off(r0), a0, b0);
        sd(rec_off(r1), a1, b1);
        const V va = cmul(a0, a1), vb = cmul(b0, b1);
        const T c = (T)rec_c(r0);
        acc0 += c * va.x;
        acc1 += c * vb.x;
        k2_visit2<3, NU, MAXU, T, HYB>(st, rec_nch(r0), va, vb, acc0, acc1, sd);
        wa += (double)acc0;
        wb += (double)acc1;
      }
    }
    mypart[(warp * 2 + 0) * 32 + lane] = wa;
    mypart[(warp * 2 + 1) * 32 + lane] = wb;
    __syncthreads();
    if (warp < 2) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + (w * 2 + warp) * 32 + lane);
      const int64_t site = tile * 64 + warp * 32 + lane;
      if (site < S) out[site] = s;
    }
  }
}

// ------------------------------------------------------- K2 (multi-output)
// Real coefficients, Re(phi), n_out outputs (BASELINE cfg5: 64): the c . A
// epilogue is a dense [sites x nodes] x [nodes x n_out] product, FP64-bound.
// Each pass handles NOC outputs with NOC accumulators per lane; every node's
// coefficient row slice is read warp-uniformly (NOC/2 LDG.128 broadcasts).
template <int NOC>
__device__ __forceinline__ void acc_row(double (&acc)[NOC], double re, const double* __restrict__ row,
                                        int stride) {
  // the coefficient rows stream from L2 in record order: pull the slice of
  // the record kPfDist ahead into L1 so this warp's next loads hit there
  constexpr int kPfDist = 4;
#pragma unroll
  for (int q = 0; q < NOC; q += 16) prefetch_l1(row + kPfDist * stride + q);
#pragma unroll
  for (int q = 0; q < NOC; q += 2) {
    const double2 c = __ldg(reinterpret_cast<const double2*>(row + q));
    acc[q] += c.x * re;
    acc[q + 1] += c.y * re;
  }
}

template <int D, int NU, int NOC, bool HYB>
__device__ __forceinline__ void k2m_visit(Stream& st, const int4* prog, int32_t cbeg, uint32_t n, double2 pv,
                                          double (&acc)[NOC], const Seeds<double, HYB>& sd,
                                          const double* __restrict__ cre, int n_out, int o0) {
  if constexpr (D > NU) {
    return;
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      const int64_t rec = cbeg + (int64_t)st.i;
      st.advance(1);
      const double2 s = sd(rec_off(r));
      if (D == NU || rec_nch(r) == 0) {
        acc_row<NOC>(acc, s.x * pv.x - s.y * pv.y, cre + rec * n_out + o0, n_out);
      } else {
        const double2 v = cmul(s, pv);
        acc_row<NOC>(acc, v.x, cre + rec * n_out + o0, n_out);
        k2m_visit<D + 1, NU, NOC, HYB>(st, prog, cbeg, rec_nch(r), v, acc, sd, cre, n_out, o0);
      }
    }
  }
}

template <int NU, int WARPS, int NOC, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_multi(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
         int Us, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
         const double* __restrict__ cre, int n_out, int o0, double* __restrict__ out,
         double2* __restrict__ gcache, double* __restrict__ part) {
  unsigned char* smem = g_smem;
  double2* sA = reinterpret_cast<double2*>(smem);
  const uint32_t rings = (uint32_t)((size_t)Us * 32 * sizeof(double2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 32 : nullptr;
  Seeds<double, HYB> sd;
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gA) + lane * 16 - (size_t)Us * 512 : nullptr;
  sd.us_bytes = (uint32_t)((size_t)Us * 512);
  const int nc = min(NOC, n_out - o0);
  double* mypart = part + (size_t)blockIdx.x * WARPS * NOC * 32;
  const int4* prog = reinterpret_cast<const int4*>(ops);
  Stream st;
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    stage_seeds<double2, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, WARPS, lane);
    __syncthreads();
    double acc[NOC];
#pragma unroll
    for (int q = 0; q < NOC; ++q) acc[q] = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(prog + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        const int64_t rec = b + (int64_t)st.i;
        st.advance(2);
        const double2 v = cmul(sd(rec_off(r0)), sd(rec_off(r1)));
        acc_row<NOC>(acc, v.x, cre + rec * n_out + o0, n_out);
        k2m_visit<3, NU, NOC, HYB>(st, prog, b, rec_nch(r0), v, acc, sd, cre, n_out, o0);
      }
    }
#pragma unroll
    for (int q = 0; q < NOC; ++q) mypart[(warp * NOC + q) * 32 + lane] = acc[q];
    __syncthreads();
    // output q is reduced by warp q % WARPS over the warps in order
    const int64_t site = tile * 32 + lane;
    for (int q = warp; q < nc; q += WARPS) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + (w * NOC + q) * 32 + lane);
      if (site < S) out[site * n_out + o0 + q] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------- K2 multi-output on DMMA
// Real coefficients, n_out outputs: the epilogue sum_k c[k][o] Re(v_k) is a
// dense [32 sites x nodes] x [nodes x n_out] GEMM per tile, issued on the
// FP64 tensor cores (mma.sync m8n8k4 f64).  Each warp stages the real parts
// of its last 8 nodes in shared memory ([8][36] doubles, lane = site); every
// 4 nodes one k-step of 4 (sites) x 4 (outputs) m8n8k4 tiles accumulates
// into registers.  Coefficient fragments are prefetched two groups ahead.
struct MmaSink {
  static constexpr int kNT = 4;       // n-tiles per pass (32 outputs)
  static constexpr int kStride = 36;  // doubles per staged node row (bank spread)
  uint32_t stg;      // g_smem byte offset of this warp's [8][kStride] staging ring
  uint32_t cnt;      // nodes stored in the current chunk
  uint32_t done;     // nodes already multiplied in (multiple of 4)
  int64_t rec0;      // global record index of the chunk's first record
  const double* cre;
  int n_out, o0, lane;
  double acc[4][kNT][2];
  double bnext[2][kNT];  // B fragments of the next two groups

  __device__ __forceinline__ void loadB(double (&b)[kNT], int64_t grp_rec) const {
    const double* row = cre + (grp_rec + (lane & 3)) * n_out + o0 + (lane >> 2);
#pragma unroll
    for (int n = 0; n < kNT; ++n) b[n] = __ldg(row + 8 * n);
  }
  __device__ __forceinline__ void begin(int64_t r0) {
    rec0 = r0;
    cnt = done = 0;
    loadB(bnext[0], rec0);
    loadB(bnext[1], rec0 + 4);
  }
  __device__ __forceinline__ void store(double re) {
    reinterpret_cast<double*>(g_smem + stg)[(cnt & 7u) * kStride + lane] = re;
    ++cnt;
  }
  // one k-step (4 nodes) once four unflushed nodes are staged; callers store
  // at most 4 nodes between calls, so at most one group is ever pending
  __device__ __forceinline__ void flush_ready() {
    if (cnt - done < 4) return;
    const double* s = reinterpret_cast<const double*>(g_smem + stg) + (done & 4u) * kStride;
    double b[kNT];
#pragma unroll
    for (int n = 0; n < kNT; ++n) {
      b[n] = bnext[0][n];
      bnext[0][n] = bnext[1][n];
    }
    loadB(bnext[1], rec0 + done + 8);
    done += 4;
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double a = s[(lane & 3) * kStride + 8 * m + (lane >> 2)];
#pragma unroll
      for (int n = 0; n < kNT; ++n)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[m][n][0]), "+d"(acc[m][n][1])
                     : "d"(a), "d"(b[n]));
    }
  }
  __device__ __forceinline__ void finish() {
    while (cnt & 3u) store(0.0);
    flush_ready();
  }
};

template <int K, bool HYB>
__device__ __forceinline__ void leaf_block_mma(const Stream& st, double2 pv, MmaSink& sk,
                                               const Seeds<double, HYB>& sd) {
  int4 r[K];
  double2 s[K];
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = st.at(j);
#pragma unroll
  for (int j = 0; j < K; ++j) s[j] = sd(rec_off(r[j]));
#pragma unroll
  for (int j = 0; j < K; ++j) sk.store(s[j].x * pv.x - s[j].y * pv.y);
}

template <int D, int NU, bool HYB>
__device__ __forceinline__ void k2mma_visit(Stream& st, uint32_t n, double2 pv, MmaSink& sk,
                                            const Seeds<double, HYB>& sd) {
  if constexpr (D > NU) {
    return;
  } else if constexpr (D == NU) {
    while (n >= 4) {
      leaf_block_mma<4, HYB>(st, pv, sk, sd);
      st.advance(4);
      n -= 4;
      sk.flush_ready();
    }
    switch (n) {
      case 1: leaf_block_mma<1, HYB>(st, pv, sk, sd); break;
      case 2: leaf_block_mma<2, HYB>(st, pv, sk, sd); break;
      case 3: leaf_block_mma<3, HYB>(st, pv, sk, sd); break;
      default: break;
    }
    st.advance(n);
    sk.flush_ready();
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      const int4 r = st.at(0);
      st.advance(1);
      const double2 v = cmul(sd(rec_off(r)), pv);
      sk.store(v.x);
      sk.flush_ready();
      k2mma_visit<D + 1, NU, HYB>(st, rec_nch(r), v, sk, sd);
    }
  }
}

template <int NU, int WARPS, bool HYB>
__global__ void __launch_bounds__(WARPS * 32, 1)
k2_mma(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label, int U,
       int Us, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
       const double* __restrict__ cre, int n_out, int o0, double* __restrict__ out,
       double2* __restrict__ gcache, double* __restrict__ part) {
  constexpr int NOC = 8 * MmaSink::kNT;
  unsigned char* smem = g_smem;
  double2* sA = reinterpret_cast<double2*>(smem);
  const uint32_t rings = (uint32_t)((size_t)Us * 32 * sizeof(double2));
  const uint32_t stgs = rings + WARPS * 64 * 16;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 32 : nullptr;
  Seeds<double, HYB> sd;
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gA) + lane * 16 - (size_t)Us * 512 : nullptr;
  sd.us_bytes = (uint32_t)((size_t)Us * 512);
  const int nc = min(NOC, n_out - o0);
  double* mypart = part + (size_t)blockIdx.x * WARPS * 32 * NOC;
  const int4* prog = reinterpret_cast<const int4*>(ops);
  Stream st;
  MmaSink sk;
  sk.stg = stgs + warp * 8 * MmaSink::kStride * 8;
  sk.cre = cre;
  sk.n_out = n_out;
  sk.o0 = o0;
  sk.lane = lane;
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    stage_seeds<double2, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, WARPS, lane);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < MmaSink::kNT; ++n) sk.acc[m][n][0] = sk.acc[m][n][1] = 0.0;
    for (int ci = warp; ci < nchunk; ci += WARPS) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(prog + b, (uint32_t)(e - b), rings + warp * 64 * 16, lane);
      sk.begin(b);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        const double2 v = cmul(sd(rec_off(r0)), sd(rec_off(r1)));
        sk.store(v.x);
        sk.store(0.0);  // the root's second record carries no coefficients
        sk.flush_ready();
        k2mma_visit<3, NU, HYB>(st, rec_nch(r0), v, sk, sd);
      }
      sk.finish();
    }
    // C fragment (m, n): rows = sites 8m + lane/4, cols = outputs 8n + 2(lane%4) + {0,1}
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int n = 0; n < MmaSink::kNT; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int site = 8 * m + (lane >> 2), o = 8 * n + 2 * (lane & 3) + j;
          mypart[((size_t)warp * 32 + site) * NOC + o] = sk.acc[m][n][j];
        }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * NOC; idx += WARPS * 32) {
      const int site_l = idx / NOC, o = idx % NOC;
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += __ldcg(mypart + ((size_t)w * 32 + site_l) * NOC + o);
      const int64_t site = tile * 32 + site_l;
      if (site < S && o < nc) out[site * n_out + o0 + o] = s;
    }
    __syncthreads();
  }
}

// ----------------------------------------------- seed gather from host rows
// The host end-to-end path: one warp per site row reads the used seed columns
// of the (page-locked, device-mapped) host table over PCIe -- consecutive
// lanes read consecutive used columns, so the runs of used labels coalesce --
// and writes the compact [S, U] table the K2 kernels then read with the
// identity slot map.  Launched on a few SMs next to the evaluation kernel.
template <typename T>
__global__ void __launch_bounds__(512) k_gather_seeds(const T* __restrict__ A, int64_t S, int L,
                                                      const int32_t* __restrict__ cols, int U, T* __restrict__ out) {
  extern __shared__ int32_t g_cols[];
  for (int i = threadIdx.x; i < U; i += blockDim.x) g_cols[i] = cols[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < S; s += nw) {
    const T* row = A + s * L;
    T* dst = out + s * U;
    for (int j0 = 0; j0 < U; j0 += 32 * 8) {
      T v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + lane + 32 * k;
        if (j < U) v[k] = __ldcs(row + g_cols[j]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = j0 + lane + 32 * k;
        if (j < U) dst[j] = v[k];
      }
    }
  }
}

// ------------------------------------------------------------- K2 (general)
// complex coefficients and/or complex output and/or several outputs: NC
// complex accumulators per lane; coefficient table [n_records, n_out].
template <int NC>
struct AccC {
  double re[NC], im[NC];
};

template <int NC>
__device__ __forceinline__ void acc_general(AccC<NC>& acc, double2 v, int64_t idx, const double* cre,
                                            const double* cim, int n_out, int o0, int nc) {
#pragma unroll
  for (int q = 0; q < NC; ++q)
    if (q < nc) {
      const double c_r = __ldg(cre + idx * n_out + o0 + q);
      const double c_i = cim ? __ldg(cim + idx * n_out + o0 + q) : 0.0;
      acc.re[q] += c_r * v.x - c_i * v.y;
      acc.im[q] += c_r * v.y + c_i * v.x;
    }
}

template <int D, int NU, int NC, bool HYB>
__device__ __forceinline__ const Op* k2g_visit(const Op* p, const Op* base, uint32_t n, double2 pv,
                                              AccC<NC>& acc, const Seeds<double, HYB>& sd,
                                              const double* cre, const double* cim, int n_out, int o0,
                                              int nc) {
  if constexpr (D > NU) {
    return p;
  } else {
    for (uint32_t j = 0; j < n; ++j) {
      OpR r = load_op(p);
      const double2 v = cmul(sd(r.off), pv);
      acc_general<NC>(acc, v, p - base, cre, cim, n_out, o0, nc);
      p = k2g_visit<D + 1, NU, NC, HYB>(p + 1, base, r.nch, v, acc, sd, cre, cim, n_out, o0, nc);
    }
    return p;
  }
}

template <int NU, int NC, bool HYB>
__global__ void __launch_bounds__(1024, 1)
k2_general(const double2* __restrict__ A, int64_t S, int L, const uint16_t* __restrict__ slot_label,
           int U, int Us, const Op* __restrict__ ops, const int32_t* __restrict__ chunk, int nchunk,
           const double* __restrict__ cre, const double* __restrict__ cim, int n_out, int o0,
           int complex_out, void* __restrict__ out, double2* __restrict__ gcache) {
  unsigned char* smem = g_smem;
  double2* sA = reinterpret_cast<double2*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)Us * 32 * sizeof(double2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 32 : nullptr;
  Seeds<double, HYB> sd;
  sd.s = (uint32_t)(lane * 16);
  sd.g = HYB ? reinterpret_cast<const char*>(gA) + lane * 16 - (size_t)Us * 512 : nullptr;
  sd.us_bytes = (uint32_t)((size_t)Us * 512);
  const int nc = min(NC, n_out - o0);
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    stage_seeds<double2, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, W, lane);
    __syncthreads();
    AccC<NC> acc;
#pragma unroll
    for (int q = 0; q < NC; ++q) acc.re[q] = acc.im[q] = 0.0;
    // static chunk assignment: warp w takes chunks w, w+W, ...
    for (int ci = warp; ci < nchunk; ci += W) {
      const Op* p = ops + chunk[ci];
      const Op* end = ops + chunk[ci + 1];
      while (p < end) {
        OpR r0 = load_op(p), r1 = load_op(p + 1);
        const double2 v = cmul(sd(r0.off), sd(r1.off));
        acc_general<NC>(acc, v, p - ops, cre, cim, n_out, o0, nc);
        p = k2g_visit<3, NU, NC, HYB>(p + 2, ops, r0.nch, v, acc, sd, cre, cim, n_out, o0, nc);
      }
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
        const int64_t site = tile * 32 + lane;
        if (site < S) {
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
  unsigned char* smem = g_smem;
  double2* sA = reinterpret_cast<double2*>(smem);
  double* red = reinterpret_cast<double*>(smem + (size_t)Us * 32 * sizeof(double2));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  double2* gA = HYB ? gcache + (size_t)blockIdx.x * (U + 1 - Us) * 32 : nullptr;
  SlotTab<HYB> tab{sA, gA, (uint32_t)Us, lane};
  const int64_t ntiles = (S + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t site = tile * 32 + lane;
    const bool valid = site < S;
    stage_seeds<double2, HYB>(A, S, L, tile, slot_label, U, Us, sA, gA, warp, W, lane);
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
