// sm_100a kernels of the evaluator.
//
//   K1  pool_*          atomic basis (pool.cuh)                          (evaluator.py:61-90)
//   K2  k2_quad         fp64 order 5-6, forward per-node products, 128-site tiles, TMEM hot rows
//       k2_mma          >= 8 real outputs: the c . A epilogue as DMMA tiles, 32-site tiles
//       k2_general      complex coefficients / complex output / 2-7 outputs, 32-site tiles
//       (k2_horner, the fp64 order <= 4 and fp32 kernel, lives in horner.cu)
//   K3  k3_naive        naive product basis, fused c . A reduction        (evaluator.py:113-121)
//   --  k_tile_seeds    tile-major seed table for k2_horner / k2_quad
//   --  k_eval_nodes    every DAG node, bit-exact (no FMA)                (evaluator.py:93-110)
//   --  k_reduce_sites  deterministic per-output site sum (energy total)
//
// The 32-site kernels (k2_mma, k2_general, k3_naive): a CTA owns a tile of
// 32 sites, lane = site; the seeds the program references are staged once per
// tile into shared memory as [slot][32 sites] (the rest in a per-CTA global
// cache), and every warp walks its own chunk of the DFS program with the
// records read warp-uniformly and the parent value of each level in
// registers.
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
// A warp-uniform value, declared so to the compiler (REDUX.OR into a uniform
// register): the program walk's control words are the same in every lane,
// and branches on them then carry no divergence bookkeeping (see horner.cu).
__device__ __forceinline__ uint32_t uni(uint32_t v) { return __reduce_or_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t rec_off(int4 r) { return (uint32_t)r.z; }
__device__ __forceinline__ uint32_t rec_nch(int4 r) { return (uint32_t)r.w & 0xFFFFu; }

// ------------------------------------------------------------ TMEM helpers
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t addr, double2 a, double2 b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(addr),
               "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)), "r"(__double2hiint(a.y)),
               "r"(__double2loint(b.x)), "r"(__double2hiint(b.x)), "r"(__double2loint(b.y)), "r"(__double2hiint(b.y)));
}

// ------------------------------------------------------ program ring (K2)
// Each warp's program ring is three 32-record slots filled by cp.async one
// block ahead; records are addressed through a running shared-memory
// pointer with immediate offsets (two mirrored records after the last slot
// keep a two-record look-ahead contiguous); block crossings are detected by
// a countdown.
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

// --------------------------------------------- tile-major seed table (K2 input)
// A [S, L] c128 -> T [ntiles][U + 1][TS] c128: row r of tile t holds slot r
// (row U = the constant ONE) for the TS sites of the tile, so the K2 kernels
// stage and fetch whole rows with coalesced loads.  Lanes walk the used
// columns in ascending order (coalesced reads of each site row); a padded
// [32][TS + 1] shared block transposes 32 columns at a time.
// cols: column of the j-th used entry (NULL: j); slots: its row (NULL: j).
// (A persistent grid over (tile, 32-column block) units, which removes the
// last-wave tail, ran 0.370 vs 0.328 ms at cfg2: a tile's column blocks on
// different CTAs at different times lose the L2 reuse of shared sectors.)
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
// serves four sites -- the per-record overhead of narrower tiles is
// amortised twice as far.  Seed rows are 2 KB ([4][32] c128): the 32 hottest
// in TMEM (16 columns per lane, one x16 load per fetch, replicated per lane
// quadrant), the next in shared memory, the tail in the per-CTA global
// cache.  24 warps x 80 registers (capi.cu kQuadWarps).
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
  // a seed of either class (inner nodes, roots): every path loads into the
  // same raw words, so the paths merge without register copies
  __device__ __forceinline__ C4 get(uint32_t off, bool hot) const {
    uint32_t t[16];
    if (hot) {
      hot_issue(off, t);
      tmem_wait_ld();
    } else {
      const uint32_t c = off * 4 - kTmemRowsQ * 2048;  // byte offset of the 2 KB cold row
      if (!HYB || c < usB) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(t[4 * k]), "=r"(t[4 * k + 1]), "=r"(t[4 * k + 2]), "=r"(t[4 * k + 3])
                       : "r"(sb + c + k * 512));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("ld.global.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(t[4 * k]), "=r"(t[4 * k + 1]), "=r"(t[4 * k + 2]), "=r"(t[4 * k + 3])
                       : "l"(gb + (c - usB) + k * 512));
      }
    }
    return unpack(t);
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

// (Round 2: the leaves summed into a chain of their own, apart from the
// node products, ran cfg4 at 405 k vs 415 k sites/s -- the single site-sum
// chain is not what binds, and the second one spills at order 6.  The Horner
// form of the leaf level -- G = sum_l c_l s_l, then Re(pv G): 8 DFMA per leaf
// instead of 12 -- ran 431 k vs 477 k: its 16-register accumulator spills.)
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
      const uint32_t w = uni((uint32_t)r.w);
      k2q_visit<D + 1, NU, MAXU, HYB>(st, w & 0xFFFFu, w >> 16, v, acc, sd, lane);
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
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5);
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
    const int cb = (int)uni((uint32_t)((int64_t)slice * nchunk / nsl)),
              ce = (int)uni((uint32_t)((int64_t)(slice + 1) * nchunk / nsl));
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
    // one partial per (chunk, site), summed in chunk order (as k2_horner)
    double* dst = whole ? mypart : tailbuf + (size_t)((it - full_tiles) / tail_parts) * nchunk * 128;
    // chunks handed out dynamically (the partials are indexed by chunk, so
    // the result does not depend on which warp ran which chunk)
    for (int ci = cb + warp; ci < ce;) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      st.begin(reinterpret_cast<const int4*>(ops) + b, uni((uint32_t)(e - b)), ring, lane);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2, lane);
        const uint32_t fl = uni((uint32_t)r1.w) >> 16, w0 = uni((uint32_t)r0.w);
        const C4 v = cmul4(sd.get((uint32_t)r0.z, fl & 1u), sd.get((uint32_t)r1.z, (fl >> 1) & 1u));
        const double c = rec_c(r0);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = __fma_rn(c, v.v[k].x, acc[k]);
        k2q_visit<3, NU, MAXU, HYB>(st, w0 & 0xFFFFu, w0 >> 16, v, acc, sd, lane);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dst[(size_t)ci * 128 + k * 32 + lane] = acc[k];
      int nx = 0;
      if (lane == 0) nx = atomicAdd(dyn, 1);
      ci = (int)uni((uint32_t)nx);  // lane 0's value (the others hold 0)
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

// ---------------------------------------------- K2 multi-output on DMMA
// Real coefficients, n_out outputs: the epilogue sum_k c[k][o] Re(v_k) is a
// dense [32 sites x nodes] x [nodes x n_out] GEMM per tile, issued on the
// FP64 tensor cores (mma.sync m8n8k4 f64).  Each warp stages the real parts
// of its last 8 nodes in shared memory ([8][36] doubles, lane = site); every
// 4 nodes one k-step of 4 (sites) x 4 (outputs) m8n8k4 tiles accumulates
// into registers.  Coefficient fragments are prefetched three groups ahead.
struct MmaSink {
  static constexpr int kNT = 4;       // n-tiles per pass (32 outputs)
  static constexpr int kStride = 36;  // doubles per staged node row (bank spread)
  uint32_t stg;      // g_smem byte offset of this warp's [8][kStride] staging ring
  uint32_t cnt;      // nodes stored in the current chunk
  uint32_t done;     // nodes already multiplied in (multiple of 4)
  int64_t rec0;      // global record index of the chunk's first record
  int64_t rec_end;   // records in the program (prefetch bound)
  const double* cre;
  int n_out, o0, lane;
  // coefficient rows this far ahead are pulled into L2 by one lane (TMA
  // bulk prefetch): the [T, n_out] matrix does not fit L2, and the two-group
  // register prefetch only covers L2 latency, not DRAM
  static constexpr int kPfRecords = 64;
  double acc[4][kNT][2];
  // coefficient groups in flight in registers (cfg5 at 2e4 sites: 2 groups
  // 220.5 k sites/s, 3 229.1 k, 4 spills: 186.2 k)
#ifndef ACEDAG_MMA_DEPTH
#define ACEDAG_MMA_DEPTH 3
#endif
  static constexpr int kDepth = ACEDAG_MMA_DEPTH;
  double bnext[kDepth][kNT];  // B fragments of the next kDepth groups

  __device__ __forceinline__ void loadB(double (&b)[kNT], int64_t grp_rec) const {
    const double* row = cre + (grp_rec + (lane & 3)) * n_out + o0 + (lane >> 2);
#pragma unroll
    for (int n = 0; n < kNT; ++n) b[n] = __ldg(row + 8 * n);
  }
  __device__ __forceinline__ void begin(int64_t r0) {
    rec0 = r0;
    cnt = done = 0;
    if (lane == 0) {  // the chunk's first rows (the flushes prefetch the rest)
      const int64_t n = rec_end - r0 < kPfRecords + 4 ? rec_end - r0 : kPfRecords + 4;
      if (n > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(cre + r0 * n_out), "r"((uint32_t)(n * n_out * 8))
                     : "memory");
    }
#pragma unroll
    for (int d = 0; d < kDepth; ++d) loadB(bnext[d], rec0 + 4 * d);
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
#pragma unroll
      for (int d = 0; d + 1 < kDepth; ++d) bnext[d][n] = bnext[d + 1][n];
    }
    loadB(bnext[kDepth - 1], rec0 + done + 4 * kDepth);
    done += 4;
    if (lane == 0) {
      const int64_t r = rec0 + done + kPfRecords;
      if (r + 4 <= rec_end)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(cre + r * n_out), "r"((uint32_t)(4 * n_out * 8))
                     : "memory");
    }
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
      k2mma_visit<D + 1, NU, HYB>(st, uni((uint32_t)r.w) & 0xFFFFu, v, sk, sd);
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
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5);
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
  sk.rec_end = __ldg(chunk + nchunk);
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
      st.begin(prog + b, uni((uint32_t)(e - b)), rings + warp * 64 * 16, lane);
      sk.begin(b);
      while (st.i < st.n) {
        const int4 r0 = st.at(0), r1 = st.at(1);
        st.advance(2);
        const double2 v = cmul(sd(rec_off(r0)), sd(rec_off(r1)));
        sk.store(v.x);
        sk.store(0.0);  // the root's second record carries no coefficients
        sk.flush_ready();
        k2mma_visit<3, NU, HYB>(st, uni((uint32_t)r0.w) & 0xFFFFu, v, sk, sd);
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
      p = k2g_visit<D + 1, NU, NC, HYB>(p + 1, base, uni(r.nch), v, acc, sd, cre, cim, n_out, o0, nc);
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
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5), W = blockDim.x >> 5;
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
        p = k2g_visit<3, NU, NC, HYB>(p + 2, ops, uni(r0.nch), v, acc, sd, cre, cim, n_out, o0, nc);
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
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5), W = blockDim.x >> 5;
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
