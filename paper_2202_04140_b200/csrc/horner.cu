// K2 Horner kernel: the recursive program evaluated bottom-up (see horner.h).
//
// Geometry: one persistent CTA per SM, 128-site tiles; lane l carries sites
// l, l+32, l+64, l+96 of the tile, so every program record serves four
// products per lane.  The seeds of a tile are split by use count: the hottest
// rows in tensor memory (fp64: 32 rows of 16 columns per lane, one
// tcgen05.ld.32x32b.x16 per fetch; fp32: 64 rows of 8 columns; replicated in
// the four lane quadrants), the next `us` rows in shared memory ([row][4][32],
// conflict-free 16-B or 8-B loads), the tail read in place from the
// tile-major table (L2).  fp64 runs 24 warps x 80 registers up to order 4
// (16 x 128 above), fp32 32 x 64 (16 above order 4): horner_warps().
//
// Per warp, the program records of a chunk stream global -> a 3-block shared
// ring (cp.async, one 512-B block per refill) whose block 0 is mirrored past
// block 2, so any 32 consecutive records from a checked position are
// readable without wrap logic; the refill check runs once per "unit" (a root
// pair, an inner record, or a deepest-level parent with its leaves), not per
// record.  The leaf loop is then: LDS.128 record, one TMEM (or four LDS)
// seed fetch, 8 FMAs.  Chunks of roots are handed to warps dynamically; each
// chunk's per-site partial is stored and the tile's partials are summed in
// chunk order by warps 0-3 at the start of the CTA's next item (double
// buffer), so a site's value does not depend on the batch, grid or split.
//
// Where the time goes (cfg2, tools/mkvariant.sh -DHX_NOFMA / -DHX_NOSEED /
// -DHX_NOGL timing builds): with the FMAs and the seed fetches both removed
// the walk alone still takes 1.29 of 2.02 ms; the FMAs add 0.45 ms, the
// global tail 0.13 ms (measured at 16 warps).  Time follows the instruction
// count at 0.5-0.6 instructions per clock per scheduler (a few in-order warps
// of dependent control code), so: the walk is declared warp-uniform to the
// compiler (uni()), which removes the divergence bookkeeping and moves the
// control state to the uniform registers -- that is what lets 24 warps fit;
// and the order-4 program sorts each root's children into same-shape runs
// that are walked by branch-free loops (run1 / run2).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "horner.h"

namespace acedag {
namespace hdev {

extern __shared__ __align__(16) unsigned char h_smem[];

// precision traits: a TMEM row holds the four sites of a lane (16 columns
// of c128, 8 of c64); a shared/global row holds the tile's 128 sites
template <typename T> struct HTr;
template <> struct HTr<double> {
  using V = double2;
  static constexpr int kCols = 16;
  static constexpr uint32_t kRow = 2048;
};
template <> struct HTr<float> {
  using V = float2;
  static constexpr int kCols = 8;
  static constexpr uint32_t kRow = 1024;
};

template <typename T>
struct C4 {
  typename HTr<T>::V v[4];
};

__device__ __forceinline__ double fmaT(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fmaT(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double mulT(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mulT(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double2 mk2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 mk2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void tmem_ld(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_ld(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
}
#ifdef HX_NOSEED
__device__ __forceinline__ void tmem_wait_ld() {}
#else
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
#endif
__device__ __forceinline__ void tmem_st8(uint32_t addr, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t a4,
                                         uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(addr), "r"(a0),
               "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7));
}
// one TMEM row: the lane's four sites
__device__ __forceinline__ void tmem_st_row(uint32_t addr, const double2 (&v)[4]) {
  tmem_st8(addr, __double2loint(v[0].x), __double2hiint(v[0].x), __double2loint(v[0].y), __double2hiint(v[0].y),
           __double2loint(v[1].x), __double2hiint(v[1].x), __double2loint(v[1].y), __double2hiint(v[1].y));
  tmem_st8(addr + 8, __double2loint(v[2].x), __double2hiint(v[2].x), __double2loint(v[2].y), __double2hiint(v[2].y),
           __double2loint(v[3].x), __double2hiint(v[3].x), __double2loint(v[3].y), __double2hiint(v[3].y));
}
__device__ __forceinline__ void tmem_st_row(uint32_t addr, const float2 (&v)[4]) {
  tmem_st8(addr, __float_as_uint(v[0].x), __float_as_uint(v[0].y), __float_as_uint(v[1].x), __float_as_uint(v[1].y),
           __float_as_uint(v[2].x), __float_as_uint(v[2].y), __float_as_uint(v[3].x), __float_as_uint(v[3].y));
}

// --------------------------------------------------- bulk copy / mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// contiguous global -> shared bulk copy on the TMA unit, completion on bar
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 r;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
// A warp-uniform value, declared so to the compiler (REDUX.OR into a uniform
// register): the walk's control words are the same in every lane, and
// branches on them then need no divergence bookkeeping (BSSY / BSYNC /
// WARPSYNC) and run on the uniform datapath.
// (cfg2: 47 -> 5 BSSY and 57 -> 1 WARPSYNC in the SASS, 126 -> 116
// registers, K2 1.945 -> 1.877 ms, fp32 1.298 -> 1.214 ms.)
__device__ __forceinline__ uint32_t uni(uint32_t v) { return __reduce_or_sync(0xffffffffu, v); }
// a record's coefficient: fp64, or (fp32 programs) the float in its low word
template <typename T>
__device__ __forceinline__ T rec_c(int4 r) {
  if constexpr (sizeof(T) == 8) return __hiloint2double(r.y, r.x);
  else return __int_as_float(r.x);
}

// ------------------------------------------------------------ program ring
// (A variant filling the slots with one lane's TMA bulk copies on per-slot
// mbarriers ran 2.25 vs 2.08 ms at cfg2, fp32 1.48 vs 1.35: the barrier waits
// and the elected-lane branch cost more than the 32-lane cp.async they save.)
struct RingH {
  static constexpr uint32_t kBlock = 512, kSpan = 3 * kBlock;
  uint32_t p;       // shared address of the next record
  uint32_t bend;    // end of the block p was in at the last check
  uint32_t base;    // slot 0
  uint32_t nslot;   // slot of the block being consumed (refilled next)
  const int4* g;    // next block to fetch
  const int4* gend;

  __device__ __forceinline__ void fetch(int lane) {
    const int4* src = g + lane;
    const bool ok = src < gend;
    const uint32_t sz = ok ? 16u : 0u;
    const int4* s = ok ? src : g;
    const uint32_t dst = base + nslot * kBlock + lane * 16;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(s), "r"(sz) : "memory");
    if (nslot == 0)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + kSpan), "l"(s), "r"(sz) : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    g += 32;
  }
  __device__ __forceinline__ void begin(const int4* gp, uint32_t len, uint32_t ring, int lane) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    g = gp;
    gend = gp + len;
    base = ring;
    p = ring;
    bend = ring + kBlock;
    nslot = 0;
    fetch(lane);
    nslot = 1;
    fetch(lane);
    nslot = 2;
    fetch(lane);
    nslot = 0;
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
  }
  __device__ __forceinline__ int4 at(uint32_t j) const { return lds128(p + j * 16); }
  // after at most 32 records since the last check
  __device__ __forceinline__ void check(int lane) {
    if (p >= bend) {
      __syncwarp();
      fetch(lane);
      nslot = nslot == 2 ? 0 : nslot + 1;
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      __syncwarp();
      bend += kBlock;
      if (bend > base + kSpan) {
        p -= kSpan;
        bend -= kSpan;
      }
    }
  }
};

// ------------------------------------------------------------------- seeds
// programs come in four copies (one per TMEM lane quadrant, the lane bits
// folded into the hot offsets) except the deep fp32 ones: at order 5-6 the
// copies (cfg4: 59 MB each against 126 MB of L2) stream from HBM, and one copy
// with the quadrant bits added per fetch runs cfg4 fp32 at 453 vs 389 k
// sites/s (fp64 at order 5-6 spills and is not the default there)
__host__ __device__ constexpr bool quad_copies(int nu, bool f32) { return nu <= 4 || !f32; }

template <typename T, bool HYB>
struct SeedsH {
  using V = typename HTr<T>::V;
  static constexpr int kC = HTr<T>::kCols;
  static constexpr uint32_t kQ = HTr<T>::kRow / 4;  // bytes between a lane's four sites in a row
  using Tm = uint32_t[kC];
  uint32_t tq;     // TMEM address of this warp's lane quadrant, column 0
  uint32_t tqo;    // added to every hot offset: 0 with per-quadrant program copies, else the lane bits
  uint32_t sb;     // shared address of cold row 0 + lane * sizeof(V)
  const char* gb;  // global tail row 0 of this tile + lane * sizeof(V)
  // z: TMEM address of the row in this warp's lane quadrant (the program
  // copy of the quadrant carries the lane bits; the allocation base is 0)
#ifdef HX_NOSEED
  __device__ __forceinline__ void hot(uint32_t z, Tm& t) const {
#pragma unroll
    for (int i = 0; i < kC; ++i) t[i] = z + i;
  }
#else
  __device__ __forceinline__ void hot(uint32_t z, Tm& t) const { tmem_ld(z + tqo, t); }
#endif
  __device__ __forceinline__ static C4<T> unpack(const Tm& t) {
    C4<T> s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (sizeof(T) == 8)
        s.v[k] = make_double2(__hiloint2double(t[4 * k + 1], t[4 * k]), __hiloint2double(t[4 * k + 3], t[4 * k + 2]));
      else
        s.v[k] = make_float2(__uint_as_float(t[2 * k]), __uint_as_float(t[2 * k + 1]));
    }
    return s;
  }
  __device__ __forceinline__ C4<T> sm(uint32_t z) const {
    C4<T> s;
#ifdef HX_NOSEED
    for (int k = 0; k < 4; ++k) s.v[k] = mk2(T(z), T(k));
    return s;
#endif
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (sizeof(T) == 8)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(s.v[k].x), "=d"(s.v[k].y) : "r"(sb + z + k * kQ));
      else
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(s.v[k].x), "=f"(s.v[k].y) : "r"(sb + z + k * kQ));
    }
    return s;
  }
  __device__ __forceinline__ C4<T> gl(uint32_t z) const {
    C4<T> s;
#ifdef HX_NOSEED
    for (int k = 0; k < 4; ++k) s.v[k] = mk2(T(z), T(k));
    return s;
#endif
#ifdef HX_NOGL
    return sm(z & 0x1FFFFu);
#endif
#pragma unroll
    for (int k = 0; k < 4; ++k) s.v[k] = __ldg(reinterpret_cast<const V*>(gb + z + k * kQ));
    return s;
  }
  // a seed of any class (roots): every path loads into the same raw words,
  // so the paths merge without register copies (cfg2 K2 1.959 -> 1.941 ms,
  // fp32 1.331 -> 1.298)
  __device__ __forceinline__ C4<T> get(uint32_t z, uint32_t cls) const {
    Tm t;
    if (cls == 0) {
      hot(z, t);
      tmem_wait_ld();
    } else if (!HYB || cls == 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if constexpr (sizeof(T) == 8)
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(t[4 * k]), "=r"(t[4 * k + 1]), "=r"(t[4 * k + 2]), "=r"(t[4 * k + 3])
                       : "r"(sb + z + k * kQ));
        else
          asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];\n" : "=r"(t[2 * k]), "=r"(t[2 * k + 1]) : "r"(sb + z + k * kQ));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if constexpr (sizeof(T) == 8)
          asm volatile("ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                       : "=r"(t[4 * k]), "=r"(t[4 * k + 1]), "=r"(t[4 * k + 2]), "=r"(t[4 * k + 3])
                       : "l"(gb + z + k * kQ));
        else
          asm volatile("ld.global.nc.v2.b32 {%0, %1}, [%2];\n" : "=r"(t[2 * k]), "=r"(t[2 * k + 1]) : "l"(gb + z + k * kQ));
      }
    }
    return unpack(t);
  }
};

template <typename T>
__device__ __forceinline__ void init_h(C4<T>& H, T c) {
#pragma unroll
  for (int k = 0; k < 4; ++k) H.v[k] = mk2(c, T(0));
}
// H += c s
template <typename T>
__device__ __forceinline__ void axpy(C4<T>& H, T c, const C4<T>& s) {
#ifdef HX_NOFMA
  H.v[0].x = fmaT(c, s.v[0].x + s.v[3].y, H.v[0].x);
  return;
#endif
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    H.v[k].x = fmaT(c, s.v[k].x, H.v[k].x);
    H.v[k].y = fmaT(c, s.v[k].y, H.v[k].y);
  }
}
// H = c + c_l s (the accumulator's first term folded into its FMAs)
template <typename T>
__device__ __forceinline__ void axpy_init(C4<T>& H, T c, T cl, const C4<T>& s) {
#ifdef HX_NOFMA
  init_h(H, c);
  H.v[0].x = fmaT(cl, s.v[0].x + s.v[3].y, c);
  return;
#endif
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    H.v[k].x = fmaT(cl, s.v[k].x, c);
    H.v[k].y = mulT(cl, s.v[k].y);
  }
}
// Hp += s H
template <typename T>
__device__ __forceinline__ void cmac(C4<T>& Hp, const C4<T>& s, const C4<T>& H) {
#ifdef HX_NOFMA
  Hp.v[0].x = fmaT(s.v[0].x + s.v[3].y, H.v[0].x, Hp.v[0].x);
  return;
#endif
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Hp.v[k].x = fmaT(s.v[k].x, H.v[k].x, Hp.v[k].x);
    Hp.v[k].y = fmaT(s.v[k].x, H.v[k].y, Hp.v[k].y);
    Hp.v[k].x = fmaT(-s.v[k].y, H.v[k].y, Hp.v[k].x);
    Hp.v[k].y = fmaT(s.v[k].y, H.v[k].x, Hp.v[k].y);
  }
}

// inner records: w = nch | nhot << 15 | nsm << 22 (children counts by class)
__device__ __forceinline__ uint32_t w_nch(uint32_t w) { return w & 0x7FFFu; }
__device__ __forceinline__ uint32_t w_nhot(uint32_t w) { return (w >> 15) & 127u; }
__device__ __forceinline__ uint32_t w_nsm(uint32_t w) { return w >> 22; }
// a node of the last inner order (its children are leaves, <= kMaxLeaves):
// w = the byte ends of its hot / shared / all leaf records past the first
// leaf, 10 bits each, so the leaf loops need no count arithmetic
__device__ __forceinline__ uint32_t lw_hot(uint32_t w) { return w & 1023u; }
__device__ __forceinline__ uint32_t lw_sm(uint32_t w) { return (w >> 10) & 1023u; }
__device__ __forceinline__ uint32_t lw_end(uint32_t w) { return w >> 20; }
constexpr uint32_t leaf_word(uint32_t n, uint32_t nh, uint32_t ns) {
  return nh * 16 | (nh + ns) * 16 << 10 | n * 16 << 20;
}
constexpr uint32_t kOneHot = leaf_word(1, 1, 0), kTwoHot = leaf_word(2, 2, 0);

// ---------------------------------------------------------------- program walk
template <uint32_t PC, typename T, bool HYB>
__device__ __forceinline__ C4<T> seed_of(const SeedsH<T, HYB>& sd, uint32_t z) {
  if constexpr (PC == 0) {
    typename SeedsH<T, HYB>::Tm t;
    sd.hot(z, t);
    tmem_wait_ld();
    return SeedsH<T, HYB>::unpack(t);
  } else if constexpr (PC == 1) {
    return sd.sm(z);
  } else {
    return sd.gl(z);
  }
}

// hot leaves [q, qh) two per TMEM round trip
template <typename T, bool HYB>
__device__ __forceinline__ void hot_leaves(uint32_t q, uint32_t qh, C4<T>& H, const SeedsH<T, HYB>& sd) {
#pragma unroll 1
  for (; q + 16 < qh; q += 32) {
    const int4 r0 = lds128(q), r1 = lds128(q + 16);
    typename SeedsH<T, HYB>::Tm t0, t1;
    sd.hot((uint32_t)r0.z, t0);
    sd.hot((uint32_t)r1.z, t1);
    tmem_wait_ld();
    axpy(H, rec_c<T>(r0), SeedsH<T, HYB>::unpack(t0));
    axpy(H, rec_c<T>(r1), SeedsH<T, HYB>::unpack(t1));
  }
  if (q < qh) {
    const int4 r = lds128(q);
    axpy(H, rec_c<T>(r), seed_of<0>(sd, (uint32_t)r.z));
  }
}

// H = c + sum over the leaves (maximum order) of one node, whose records
// start at q (first: l, already read): hot, shared, global -- at most
// kMaxLeaves, so they lie in the checked ring window.  The first leaf's FMA
// carries c; a node whose leaves are all hot (the usual case) skips the
// other loops.
template <typename T, bool HYB>
__device__ __forceinline__ void leaves(uint32_t q, uint32_t w, T c, int4 l, C4<T>& H, const SeedsH<T, HYB>& sd) {
  const uint32_t qh = q + lw_hot(w), qs = q + lw_sm(w), qe = q + lw_end(w);
  if (qh != q) {
    axpy_init(H, c, rec_c<T>(l), seed_of<0>(sd, (uint32_t)l.z));
    hot_leaves(q + 16, qh, H, sd);
    if (qh == qe) return;
    q = qh;
  } else if (qe != q) {
    axpy_init(H, c, rec_c<T>(l), qs != q ? sd.sm((uint32_t)l.z) : sd.gl((uint32_t)l.z));
    q += 16;
  } else {
    init_h(H, c);
    return;
  }
#pragma unroll 1
  for (; q < qs; q += 16) {
    const int4 r = lds128(q);
    axpy(H, rec_c<T>(r), sd.sm((uint32_t)r.z));
  }
  if constexpr (HYB) {
#pragma unroll 1
    for (; q < qe; q += 16) {
      const int4 r = lds128(q);
      axpy(H, rec_c<T>(r), sd.gl((uint32_t)r.z));
    }
  }
}

// n sibling nodes of order NU-1 whose seeds are of class PC; each adds
// s * (c + sum_leaves c_l s_l) to Hp.  The node record and the one after it
// (its first leaf) are read together; for the commonest shapes (one or two
// hot leaves) the leaf seeds and a hot node seed share one TMEM round trip.
template <uint32_t PC, bool RUNS, typename T, bool HYB>
__device__ __forceinline__ void parents(RingH& st, uint32_t n, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane) {
  using SD = SeedsH<T, HYB>;
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const int4 r = st.at(0), l = st.at(1);
    const uint32_t w = uni((uint32_t)r.w);
    C4<T> H, sp;
    if (!RUNS && w == kOneHot) {
      typename SD::Tm tl;
      sd.hot((uint32_t)l.z, tl);
      if constexpr (PC == 0) {
        typename SD::Tm tp;
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SD::unpack(tp);
      } else {
        tmem_wait_ld();
      }
      axpy_init(H, rec_c<T>(r), rec_c<T>(l), SD::unpack(tl));
    } else if (!RUNS && w == kTwoHot) {
      const int4 l2 = st.at(2);
      typename SD::Tm tl, tl2;
      sd.hot((uint32_t)l.z, tl);
      sd.hot((uint32_t)l2.z, tl2);
      if constexpr (PC == 0) {
        typename SD::Tm tp;
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SD::unpack(tp);
      } else {
        tmem_wait_ld();
      }
      axpy_init(H, rec_c<T>(r), rec_c<T>(l), SD::unpack(tl));
      axpy(H, rec_c<T>(l2), SD::unpack(tl2));
    } else {
      leaves(st.p + 16, w, rec_c<T>(r), l, H, sd);
      if constexpr (PC == 0) sp = seed_of<0>(sd, (uint32_t)r.z);
    }
    if constexpr (PC != 0) sp = seed_of<PC>(sd, (uint32_t)r.z);
    cmac(Hp, sp, H);
    st.p += 16 + lw_end(w);
    st.check(lane);
  }
}

// ---- shape-sorted runs (order-4 programs) --------------------------------
// The walk is bound by its own control chain (record load -> compare ->
// branch -> next address; ~140 cycles per record per warp with the FMAs and
// seed fetches removed), so the commonest node shapes get loops with no
// data-dependent branch: the order-3 children of a root are sorted, inside
// each seed class, into S1 (exactly one leaf, hot), S2 (exactly two leaves,
// both hot) and the rest; the root's second record carries the six run
// lengths.  An S1 node is the two records {c, z, .}{c_l, z_l, .}, an S2 node
// three; up to 32 records (the checked ring window) go between ring checks,
// and S1 nodes are taken two at a time so that four seed fetches are in
// flight behind one wait.
template <uint32_t PC, typename T, bool HYB>
__device__ __forceinline__ void run1(RingH& st, uint32_t n, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane) {
  using SD = SeedsH<T, HYB>;
#pragma unroll 1
  while (n) {
    const uint32_t m = n < 16u ? n : 16u;
    n -= m;
    uint32_t q = st.p;
    const uint32_t qe = q + m * 32u;
#pragma unroll 1
    for (; q < qe; q += 32) {
      const int4 r = lds128(q), l = lds128(q + 16);
      typename SD::Tm tl;
      sd.hot((uint32_t)l.z, tl);
      C4<T> sp, H;
      if constexpr (PC == 0) {
        typename SD::Tm tp;
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SD::unpack(tp);
      } else {
        sp = seed_of<PC>(sd, (uint32_t)r.z);
        tmem_wait_ld();
      }
      axpy_init(H, rec_c<T>(r), rec_c<T>(l), SD::unpack(tl));
      cmac(Hp, sp, H);
    }
    st.p = qe;
    st.check(lane);
  }
}

template <uint32_t PC, typename T, bool HYB>
__device__ __forceinline__ void run2(RingH& st, uint32_t n, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane) {
  using SD = SeedsH<T, HYB>;
#pragma unroll 1
  while (n) {
    const uint32_t m = n < 10u ? n : 10u;
    n -= m;
    uint32_t q = st.p;
    const uint32_t qe = q + m * 48u;
#pragma unroll 1
    for (; q < qe; q += 48) {
      const int4 r = lds128(q), l = lds128(q + 16), l2 = lds128(q + 32);
      typename SD::Tm tl, tl2;
      sd.hot((uint32_t)l.z, tl);
      sd.hot((uint32_t)l2.z, tl2);
      C4<T> sp, H;
      if constexpr (PC == 0) {
        typename SD::Tm tp;
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SD::unpack(tp);
      } else {
        sp = seed_of<PC>(sd, (uint32_t)r.z);
        tmem_wait_ld();
      }
      axpy_init(H, rec_c<T>(r), rec_c<T>(l), SD::unpack(tl));
      axpy(H, rec_c<T>(l2), SD::unpack(tl2));
      cmac(Hp, sp, H);
    }
    st.p = qe;
    st.check(lane);
  }
}

template <int D, int NU, typename T, bool HYB>
__device__ __forceinline__ void children(RingH& st, uint32_t w, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane);

// n sibling nodes of order D < NU-1 with seeds of class PC
template <int D, int NU, uint32_t PC, typename T, bool HYB>
__device__ __forceinline__ void inner(RingH& st, uint32_t n, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane) {
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const int4 r = st.at(0);
    st.p += 16;
    st.check(lane);
    C4<T> H;
    init_h(H, rec_c<T>(r));
    children<D + 1, NU>(st, uni((uint32_t)r.w), H, sd, lane);
    cmac(Hp, seed_of<PC>(sd, (uint32_t)r.z), H);
  }
}

// the children (order D) of a node whose accumulator is Hp, by seed class;
// the ring was checked right before the first child record
template <int D, int NU, typename T, bool HYB>
__device__ __forceinline__ void children(RingH& st, uint32_t w, C4<T>& Hp, const SeedsH<T, HYB>& sd, int lane) {
  const uint32_t nh = w_nhot(w), ns = w_nsm(w), ng = w_nch(w) - nh - ns;
  if constexpr (D == NU - 1) {
    parents<0, false>(st, nh, Hp, sd, lane);
    parents<1, false>(st, ns, Hp, sd, lane);
    if (HYB) parents<2, false>(st, ng, Hp, sd, lane);
  } else if constexpr (D < NU - 1) {
    inner<D, NU, 0>(st, nh, Hp, sd, lane);
    inner<D, NU, 1>(st, ns, Hp, sd, lane);
    if (HYB) inner<D, NU, 2>(st, ng, Hp, sd, lane);
  }
}

template <int NU, typename T, bool HYB>
__device__ __forceinline__ void root(RingH& st, double (&acc)[4], const SeedsH<T, HYB>& sd, int lane) {
  const int4 r0 = st.at(0), r1 = st.at(1);
  const T c = rec_c<T>(r0);
  const uint32_t fl = uni((uint32_t)r1.w);
  if (fl & 16u) {
    // an order-1 coefficient: phi += c Re(s_a), no children
    const C4<T> sa = sd.get((uint32_t)r0.z, fl & 3u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (sizeof(T) == 8) acc[k] = __fma_rn(sa.v[k].x, c, acc[k]);
      else acc[k] += (double)mulT(sa.v[k].x, c);
    }
    st.p += 32;
    st.check(lane);
    return;
  }
  C4<T> H;
  if constexpr (NU == 3) {
    const uint32_t w3 = uni((uint32_t)r0.w);
    leaves(st.p + 32, w3, c, st.at(2), H, sd);
    st.p += 32 + lw_end(w3);
    st.check(lane);
  } else {
    init_h(H, c);
    st.p += 32;
    st.check(lane);
    if constexpr (NU == 4) {
      // run lengths of the class-and-shape-sorted children: r0.w = the general
      // runs (hot | shared << 10 | global << 20); r1.x / r1.y = S1 | S2 << 16
      // of the hot / shared classes; r1.w >> 8 = S1 | S2 << 12 of the global one
      const uint32_t wg = uni((uint32_t)r0.w), wh = uni((uint32_t)r1.x), ws = uni((uint32_t)r1.y);
      run1<0>(st, wh & 0xFFFFu, H, sd, lane);
      run2<0>(st, wh >> 16, H, sd, lane);
      parents<0, true>(st, wg & 1023u, H, sd, lane);
      if (ws | (wg & 0xFFC00u)) {
        run1<1>(st, ws & 0xFFFFu, H, sd, lane);
        run2<1>(st, ws >> 16, H, sd, lane);
        parents<1, true>(st, (wg >> 10) & 1023u, H, sd, lane);
      }
      if (HYB && (fl >> 8 | wg >> 20)) {
        run1<2>(st, (fl >> 8) & 0xFFFu, H, sd, lane);
        run2<2>(st, fl >> 20, H, sd, lane);
        parents<2, true>(st, wg >> 20, H, sd, lane);
      }
    } else if constexpr (NU > 4) {
      children<3, NU>(st, uni((uint32_t)r0.w), H, sd, lane);
    }
  }
  // (a branch-free form -- three predicated load groups into the same
  // registers -- spilled and ran 2.42 vs 1.96 ms at cfg2)
  const C4<T> sa = sd.get((uint32_t)r0.z, fl & 3u), sb = sd.get((uint32_t)r1.z, (fl >> 2) & 3u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const T abx = fmaT(sa.v[k].x, sb.v[k].x, -mulT(sa.v[k].y, sb.v[k].y));
    const T aby = fmaT(sa.v[k].x, sb.v[k].y, mulT(sa.v[k].y, sb.v[k].x));
    if constexpr (sizeof(T) == 8) {
      acc[k] = __fma_rn(abx, H.v[k].x, acc[k]);
      acc[k] = __fma_rn(-aby, H.v[k].y, acc[k]);
    } else {  // the site's sum over roots in fp64
      acc[k] += (double)fmaT(abx, H.v[k].x, -mulT(aby, H.v[k].y));
    }
  }
}

// Tab: tile-major seed table [ntiles][U + 1][128] (c128 or c64)
template <int NU, typename T, bool HYB, int W>
__global__ void __launch_bounds__(W * 32, 1)
k2_horner(const typename HTr<T>::V* __restrict__ Tab, int64_t S, int U, int us, const OpH* __restrict__ ops,
          const int32_t* __restrict__ chunk, const int32_t* __restrict__ croots, int nchunk,
          double* __restrict__ out, double* __restrict__ part, int64_t full_tiles, int tail_parts,
          double* __restrict__ tailbuf) {
  using V = typename HTr<T>::V;
  constexpr int kC = HTr<T>::kCols;
  constexpr uint32_t kRow = HTr<T>::kRow;
  constexpr int kHot = 512 / kC;
  unsigned char* smem = h_smem;
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5);
  const int rows = U + 1;  // table rows (row U: the constant ONE, unused here)
  const int hot = U < kHot ? U : kHot;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t rings = sbase + (uint32_t)us * kRow;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + (size_t)us * kRow + W * kHornerRing);
  int* dyn = reinterpret_cast<int*>(tslot) + 1;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(tslot) + 8;  // bulk-copy completion (8 B aligned)
  uint32_t bar_phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tbase = *tslot;
  if (tbase != 0) __trap();  // the program's TMEM addresses assume the whole TMEM at column 0
  SeedsH<T, HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.tqo = quad_copies(NU, sizeof(T) == 4) ? 0u : sd.tq;
  sd.sb = sbase + (uint32_t)(lane * sizeof(V));
  sd.gb = nullptr;
  const uint32_t ring = rings + (uint32_t)warp * kHornerRing;
  const int32_t nops = __ldg(chunk + nchunk);  // records per quadrant copy
  // two partial buffers: a whole tile's chunk partials are summed by warps
  // 0-3 at the start of the CTA's next item (hidden by the dynamic chunk
  // hand-out) instead of in a barrier bubble at the tile end
  double* mypart0 = part + (size_t)blockIdx.x * nchunk * 128 * 2;
  int pbuf = 0;
  int64_t pend_tile = -1;
  auto sum_tile = [&](int64_t t, const double* src) {
    const int i = threadIdx.x;  // warps 0-3: site t * 128 + i
    double s = 0.0;
#pragma unroll 16
    for (int ci = 0; ci < nchunk; ++ci) s += __ldcg(src + (size_t)ci * 128 + i);
    const int64_t site = t * 128 + i;
    if (site < S) out[site] = s;
  };
  RingH st;
  const int64_t ntiles = (S + 127) / 128;
  const int64_t nitems = full_tiles + (ntiles - full_tiles) * tail_parts;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const bool whole = it < full_tiles;
    const int64_t tile = whole ? it : full_tiles + (it - full_tiles) / tail_parts;
    const int slice = whole ? 0 : (int)((it - full_tiles) % tail_parts);
    const int nsl = whole ? 1 : tail_parts;
    const int cb = (int)uni((uint32_t)((int64_t)slice * nchunk / nsl)),
              ce = (int)uni((uint32_t)((int64_t)(slice + 1) * nchunk / nsl));
    const V* Tt = Tab + tile * (int64_t)rows * 128;
    // the next item's on-chip rows into L2 while this tile computes (also
    // prefetching this tile's cold tail ran 2.09 vs 2.06 ms: L2 thrash)
    if (threadIdx.x == 0 && it + gridDim.x < nitems) {
      const int64_t nit = it + gridDim.x;
      const int64_t nt = nit < full_tiles ? nit : full_tiles + (nit - full_tiles) / tail_parts;
      if (nt != tile) {
        const char* src = reinterpret_cast<const char*>(Tab + nt * (int64_t)rows * 128);
        const uint32_t bytes = (uint32_t)(hot + us) * kRow;
        for (uint32_t o = 0; o < bytes; o += 32768u) {
          const uint32_t n = bytes - o < 32768u ? bytes - o : 32768u;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src + o), "r"(n) : "memory");
        }
      }
    }
    // shared rows: the tile's us rows are contiguous in the table, so one
    // elected thread moves them with TMA bulk copies (cp.async.bulk, 64 KB
    // pieces) completing on an mbarrier while the warps fill TMEM below; the
    // previous item's generic reads of these rows ended at its barrier
    if (threadIdx.x == 0 && us > 0) {
      const char* src = reinterpret_cast<const char*>(Tt + (size_t)hot * 128);
      const uint32_t bytes = (uint32_t)us * kRow;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      mbar_expect_tx(bar, bytes);
      for (uint32_t o = 0; o < bytes; o += 65536u)
        bulk_g2s(sbase + o, src + o, bytes - o < 65536u ? bytes - o : 65536u, bar);
    }
    if (HYB) sd.gb = reinterpret_cast<const char*>(Tt + (size_t)(hot + us) * 128) + lane * sizeof(V);
    // TMEM rows: each lane quadrant's W/4 warps write all hot rows
    for (int h0 = warp >> 2; h0 < hot; h0 += 4 * (W / 4)) {
      V v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (W / 4);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[q][k] = h < hot ? ld_stream(Tt + (size_t)h * 128 + k * 32 + lane) : mk2(T(0), T(0));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (W / 4);
        if (h < hot) tmem_st_row(sd.tq + (uint32_t)(h * kC), v[q]);
      }
    }
    if (us > 0) {
      mbar_wait(bar, bar_phase);
      bar_phase ^= 1;
    }
    if (threadIdx.x == 0) *dyn = cb + W;
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (pend_tile >= 0 && warp < 4) sum_tile(pend_tile, mypart0 + (size_t)(pbuf ^ 1) * nchunk * 128);
    double* mypart = mypart0 + (size_t)pbuf * nchunk * 128;
    double* dst = whole ? mypart : tailbuf + (size_t)((it - full_tiles) / tail_parts) * nchunk * 128;
    for (int ci = cb + warp; ci < ce;) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      const int32_t nr = (int32_t)uni((uint32_t)__ldg(croots + ci));
      st.begin(reinterpret_cast<const int4*>(ops) + (quad_copies(NU, sizeof(T) == 4) ? (size_t)(warp & 3) * nops : (size_t)0) + b,
               (uint32_t)(e - b), ring, lane);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int32_t k = 0; k < nr; ++k) root<NU>(st, acc, sd, lane);
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
    pend_tile = whole ? tile : -1;
    if (whole) pbuf ^= 1;
  }
  if (pend_tile >= 0 && warp < 4) sum_tile(pend_tile, mypart0 + (size_t)(pbuf ^ 1) * nchunk * 128);
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

}  // namespace hdev

// ------------------------------------------------------------------- host
// warps per CTA.  fp64, order <= 4: 24 x 80 registers since the walk is
// declared warp-uniform (the uniform datapath took the control state out of
// the vector registers: 126 -> 116 unconstrained, and at 80 ptxas spills only
// three of the four site sums, touched once per root): cfg2 K2 1.877 -> 1.776
// ms.  (20 warps x 96 registers: 2.49 ms -- 228 B of spills inside the loops;
// 28 x 72: 2.17 ms; 32 x 64: 2.81 ms.  Before the uniform walk 20 and 24
// warps ran 7% / 17% slower than 16.)  fp64 above order 4: 16.  fp32: 32 for
// order <= 4 (64 registers; 1.39 vs 1.58 ms at 16, cfg2), 16 above (one more
// accumulator per level; 20 ran 611 vs 528 ms at cfg4).  ACEDAG_HWARPS32 = 16
// | 32 overrides for fp32.
int horner_warps(bool f32, int nu) {
  static int w32 = [] {
    const char* e = getenv("ACEDAG_HWARPS32");
    const int v = e ? atoi(e) : 0;
    return v == 16 || v == 32 ? v : 0;
  }();
  // (fp64 order 5-6 at 12 warps / 170 registers -- no spills -- still ran
  // cfg4 at 150 k vs 415 k sites/s for k2_quad: the deep inner levels, not
  // the registers, are what make Horner slow there; k2_quad stays)
  if (!f32) return nu <= 4 ? kHornerWarps : 16;
  if (w32) return w32;
  return nu <= 4 ? 32 : 16;
}

int horner_us_max(size_t smem_optin, bool f32, int nu) {
  const size_t fixed = (size_t)horner_warps(f32, nu) * kHornerRing + 16;
  return smem_optin > fixed ? (int)((smem_optin - fixed) / horner_row_bytes(f32)) : 0;
}
size_t horner_smem(int us, bool f32, int nu) {
  return (size_t)us * horner_row_bytes(f32) + (size_t)horner_warps(f32, nu) * kHornerRing + 16;
}

namespace {
// relative size of the second half of the chunks (ACEDAG_HGUIDE; 1 = equal)
double guided_tail() {
  static double v = [] {
    const char* e = getenv("ACEDAG_HGUIDE");
    const double x = e ? atof(e) : 1.0;
    return x > 0 ? x : 1.0;
  }();
  return v;
}
// extra chunk-cost weight of a shared-memory / global-tail seed fetch (a
// record costs 1 (leaf) or cost_w(1) (node), a root unit cost_w(2) more);
// measured at cfg2 (node, root, shared, global): (3, 2, 0, 0) 2.115 ms,
// (3, 2, 1, 10) 2.081, (2, 4, 0.5, 8) 2.071, (3, 8, 1, 10) 2.102 -- a chunk's
// real time follows its L2 fetches.  Re-tuned for the 24-warp kernel with
// same-shape runs: (1.5, 8, 2, 8) 1.729 ms vs (2, 4, 0.5, 8) 1.754.
// ACEDAG_HCOST_S / ACEDAG_HCOST_G override.
// record weights: [1] a node record (leaf = 1), [2] extra per root unit
// (ACEDAG_HCOST_N / ACEDAG_HCOST_R)
double cost_w(int which) {
  static double wn = [] { const char* e = getenv("ACEDAG_HCOST_N"); return e ? atof(e) : 1.5; }();
  static double wr = [] { const char* e = getenv("ACEDAG_HCOST_R"); return e ? atof(e) : 8.0; }();
  return which == 1 ? wn : wr;
}
double class_cost(uint8_t cls) {
  static double ws = [] { const char* e = getenv("ACEDAG_HCOST_S"); return e ? atof(e) : 2.0; }();
  static double wg = [] { const char* e = getenv("ACEDAG_HCOST_G"); return e ? atof(e) : 8.0; }();
  return cls == 1 ? ws : (cls == 2 ? wg : 0.0);
}
struct HornerEnc {
  const PlanHost& H;
  uint32_t hot, us, U;
  int nu;
  std::vector<OpH>& out;
  uint32_t hot_cols, row_bytes;  // TMEM columns per hot row, bytes per shared/global row
  std::vector<uint8_t> hot_rec;  // record's z is a TMEM column (gets the lane-quadrant bits per copy)
  std::vector<uint8_t> cls_rec;  // seed class of each record (chunk cost model)
  bool ok = true;

  uint32_t cls(uint32_t s) const { return s < hot ? 0u : (s < hot + us ? 1u : 2u); }
  uint32_t zof(uint32_t s) const {
    const uint32_t c = cls(s);
    return c == 0 ? s * hot_cols : (c == 1 ? (s - hot) * row_bytes : (s - hot - us) * row_bytes);
  }
  static uint32_t slot(const Op& o) { return o.off / kRowBytes; }
  size_t skip(size_t pos) const {
    size_t q = pos + 1;
    for (uint32_t j = 0; j < H.ops[pos].nch; ++j) q = skip(q);
    return q;
  }
  void count(uint32_t c, uint32_t k, uint32_t& n, uint32_t& nh, uint32_t& ns) {
    n += k;
    if (c == 0) nh += k;
    if (c == 1) ns += k;
  }
  uint32_t pack(uint32_t n, uint32_t nh, uint32_t ns) {
    if (n > 0x7FFFu || nh > 127u || ns > 1023u) ok = false;
    return n | nh << 15 | ns << 22;
  }
  // leaves [first, first + n) of a node (positions of records with nch = 0)
  void emit_leaves(const std::vector<size_t>& kids, size_t b, size_t e) {
    for (size_t j = b; j < e; ++j) {
      const Op& l = H.ops[kids[j]];
      out.push_back(OpH{l.c, zof(slot(l)), 0u});
      hot_rec.push_back(cls(slot(l)) == 0);
      cls_rec.push_back((uint8_t)cls(slot(l)));
    }
  }
  // the record word of a node whose children are leaves (hdev::leaf_word)
  uint32_t leaf_w(const std::vector<size_t>& kids, size_t b, size_t e) {
    uint32_t n = 0, nh = 0, ns = 0;
    for (size_t j = b; j < e; ++j) count(cls(slot(H.ops[kids[j]])), 1, n, nh, ns);
    return hdev::leaf_word(n, nh, ns);
  }
  std::vector<size_t> kids_of(size_t pos) const { return kids_from(pos + 1, H.ops[pos].nch); }
  std::vector<size_t> kids_from(size_t q, uint32_t n) const {
    std::vector<size_t> k;
    for (uint32_t j = 0; j < n; ++j) {
      k.push_back(q);
      q = skip(q);
    }
    return k;
  }
  // the node at pos (order d >= 3); returns the records emitted at its own
  // level (a node of order nu-1 with more than kMaxLeaves leaves becomes
  // several copies of one seed: the first carries c, each a slice of leaves)
  uint32_t node(size_t pos, int d) {
    const Op& o = H.ops[pos];
    const uint32_t z = zof(slot(o));
    const std::vector<size_t> kids = kids_of(pos);
    const uint8_t zh = cls(slot(o)) == 0, zc = (uint8_t)cls(slot(o));
    if (d == nu) {
      out.push_back(OpH{o.c, z, 0u});
      hot_rec.push_back(zh);
      cls_rec.push_back(zc);
      return 1;
    }
    if (d == nu - 1) {
      uint32_t copies = 0;
      size_t b = 0;
      do {
        const size_t e = std::min(kids.size(), b + kMaxLeaves);
        out.push_back(OpH{b == 0 ? o.c : 0.0, z, leaf_w(kids, b, e)});
        hot_rec.push_back(zh);
        cls_rec.push_back(zc);
        emit_leaves(kids, b, e);
        copies++;
        b = e;
      } while (b < kids.size());
      return copies;
    }
    const size_t me = out.size();
    out.push_back(OpH{o.c, z, 0u});
    hot_rec.push_back(zh);
    cls_rec.push_back(zc);
    uint32_t n = 0, nh = 0, ns = 0;
    for (size_t k : kids) count(cls(slot(H.ops[k])), node(k, d + 1), n, nh, ns);
    out[me].w = pack(n, nh, ns);
    return 1;
  }
  // a root at pos (two records); returns the position past its subtree
  size_t root(size_t pos) {
    const Op& a = H.ops[pos];
    const Op& b = H.ops[pos + 1];
    const uint32_t sa = slot(a), sb = slot(b);
    const bool single = sb == U;
    const uint32_t fl = cls(sa) | (single ? 0u : cls(sb)) << 2 | (single ? 16u : 0u);
    std::vector<size_t> kids = kids_from(pos + 2, a.nch);  // children follow the pair
    if (nu == 3) {
      size_t bb = 0;
      bool first = true;
      do {
        const size_t e = std::min(kids.size(), bb + kMaxLeaves);
        out.push_back(OpH{first ? a.c : 0.0, zof(sa), leaf_w(kids, bb, e)});
        out.push_back(OpH{0.0, single ? 0u : zof(sb), fl});
        hot_rec.push_back(cls(sa) == 0);
        hot_rec.push_back(!single && cls(sb) == 0);
        cls_rec.push_back((uint8_t)cls(sa));
        cls_rec.push_back((uint8_t)(single ? 0 : cls(sb)));
        emit_leaves(kids, bb, e);
        nroots++;
        first = false;
        bb = e;
      } while (bb < kids.size());
    } else {
      const size_t me = out.size();
      out.push_back(OpH{a.c, zof(sa), 0u});
      out.push_back(OpH{0.0, single ? 0u : zof(sb), fl});
      hot_rec.push_back(cls(sa) == 0);
      hot_rec.push_back(!single && cls(sb) == 0);
      cls_rec.push_back((uint8_t)cls(sa));
      cls_rec.push_back((uint8_t)(single ? 0 : cls(sb)));
      uint32_t n = 0, nh = 0, ns = 0;
      if (nu == 4) {
        // shape-sorted runs: per class S1 (one hot leaf), S2 (two hot leaves), the rest
        auto shape = [&](size_t k) -> uint32_t {
          const std::vector<size_t> lv = kids_of(k);
          if (lv.empty() || lv.size() > 2) return 2u;
          for (size_t q : lv)
            if (cls(slot(H.ops[q])) != 0) return 2u;
          return (uint32_t)lv.size() - 1u;
        };
        std::stable_sort(kids.begin(), kids.end(), [&](size_t a, size_t b) {
          const uint32_t ca = cls(slot(H.ops[a])), cb = cls(slot(H.ops[b]));
          return ca != cb ? ca < cb : shape(a) < shape(b);
        });
        runs4 = {};
        for (size_t k : kids) {
          const uint32_t sh = shape(k);
          if (sh < 2) runs4.r[cls(slot(H.ops[k]))][sh]++;
        }
      }
      for (size_t k : kids) count(cls(slot(H.ops[k])), node(k, 3), n, nh, ns);
      out[me].w = pack(n, nh, ns);
      if (nu == 4) {
        // order-4 roots carry run lengths instead (see hdev::root): general
        // runs in r0.w, S1 / S2 runs in the second record's free fields
        const uint32_t byc[3] = {nh, ns, n - nh - ns};
        uint32_t gen[3];
        for (int c = 0; c < 3; ++c) {
          gen[c] = byc[c] - runs4.r[c][0] - runs4.r[c][1];
          if (gen[c] > 1023u || runs4.r[c][0] > 4095u || runs4.r[c][1] > 4095u) ok = false;
        }
        out[me].w = gen[0] | gen[1] << 10 | gen[2] << 20;
        out[me + 1].w |= runs4.r[2][0] << 8 | runs4.r[2][1] << 20;
        const uint64_t bits = (uint64_t)(runs4.r[0][0] | runs4.r[0][1] << 16) |
                              (uint64_t)(runs4.r[1][0] | runs4.r[1][1] << 16) << 32;
        run_bits.emplace_back(me + 1, bits);
      }
      nroots++;
    }
    size_t q = pos + 2;
    for (size_t j = 0; j < kids.size(); ++j) q = skip(q);
    return q;
  }
  int32_t nroots = 0;
  struct Runs4 { uint32_t r[3][2]; } runs4{};
  // (record index, packed run lengths) of the roots' second records (order 4):
  // written into the coefficient field after the fp32 coefficient conversion
  std::vector<std::pair<size_t, uint64_t>> run_bits;
};
}  // namespace

bool encode_horner(const PlanHost& H, bool f32, uint32_t hot, uint32_t us, std::vector<OpH>& out,
                   std::vector<int32_t>& chunk, std::vector<int32_t>& croots, bool four_copies) {
  out.clear();
  const size_t nchunk = H.chunk.size() > 0 ? H.chunk.size() - 1 : 0;
  HornerEnc E{H, hot, us, (uint32_t)H.slot_label.size(), H.max_order, out, f32 ? 8u : 16u,
              (uint32_t)horner_row_bytes(f32)};
  // every root unit (a split root is several), with its record offset and cost
  std::vector<size_t> start;
  std::vector<double> cost;
  {
    size_t i = 0;
    while (i < H.ops.size()) {
      const size_t b0 = out.size();
      const int32_t r0 = E.nroots;
      i = E.root(i);
      // the units the root became (a split NU=3 root: consecutive pair + leaves)
      size_t q = b0;
      for (int32_t k = r0; k < E.nroots; ++k) {
        // a split order-3 root is its pair + leaves (leaf word: n leaves at w >> 24)
        const size_t e = E.nroots - r0 == 1 ? out.size() : q + 2 + (out[q].w >> 24);
        start.push_back(q);
        double c = cost_w(2);
        for (size_t t = q; t < e; ++t)
          c += ((t != q + 1 && out[t].w) ? cost_w(1) : 1.0) + class_cost(E.cls_rec[t]);
        cost.push_back(c);
        q = e;
      }
    }
  }
  // guided chunking: the first half of the chunks take a share `big` of the
  // work each, the second half a quarter of that, so the last chunks a warp
  // grabs in a tile are short and the tile-end barrier waits less
  const size_t nu = start.size();
  double total = 0;
  for (double c : cost) total += c;
  std::vector<double> wt(nchunk);
  double wsum = 0;
  for (size_t i = 0; i < nchunk; ++i) wsum += (wt[i] = i < nchunk / 2 ? 1.0 : guided_tail());
  chunk.assign(nchunk + 1, (int32_t)out.size());
  croots.assign(nchunk, 0);
  chunk[0] = 0;
  size_t u = 0;
  double acc = 0, target = 0;
  for (size_t ci = 0; ci < nchunk; ++ci) {
    chunk[ci] = (int32_t)(u < nu ? start[u] : out.size());
    target += wt[ci] / wsum * total;
    int32_t nr = 0;
    while (u < nu && (acc + 0.5 * cost[u] <= target || ci + 1 == nchunk)) {
      acc += cost[u++];
      nr++;
    }
    croots[ci] = nr;
  }
  chunk[nchunk] = (int32_t)out.size();
  // one copy per TMEM lane quadrant: a TMEM column offset carries the
  // quadrant's lane bits, so a hot fetch is R2UR + tcgen05.ld with no add
  const size_t n = out.size();
  if (E.hot_rec.size() != n) return false;
  if (f32)  // fp32 programs carry each coefficient as a float in the low word
    for (OpH& o : out) {
      const float f = (float)o.c;
      uint32_t b;
      std::memcpy(&b, &f, 4);
      const uint64_t u = b;
      std::memcpy(&o.c, &u, 8);
    }
  for (const auto& rb : E.run_bits) std::memcpy(&out[rb.first].c, &rb.second, 8);
  if (!four_copies && !hdev::quad_copies(H.max_order, f32)) return E.ok && n < (size_t)INT32_MAX;
  out.resize(4 * n);
  for (size_t q = 1; q < 4; ++q)
    for (size_t i = 0; i < n; ++i) {
      out[q * n + i] = out[i];
      if (E.hot_rec[i]) out[q * n + i].z += (uint32_t)(q * 32) << 16;
    }
  return E.ok && 4 * n < (size_t)INT32_MAX;
}

template <int NU, typename T, bool HYB>
static cudaError_t launch_nu(const void* Tab, int64_t S, int U, int us, const OpH* ops, const int32_t* chunk,
                             const int32_t* croots, int nchunk, double* out, double* part, int64_t full, int parts,
                             double* tail, int grid, cudaStream_t st) {
  const int W = horner_warps(sizeof(T) == 4, NU);
  auto k = hdev::k2_horner<NU, T, HYB, 16>;
  if constexpr (sizeof(T) == 8 && NU <= 4) k = hdev::k2_horner<NU, T, HYB, kHornerWarps>;
  if constexpr (sizeof(T) == 4) {
    if (W == 32) k = hdev::k2_horner<NU, T, HYB, 32>;
  }
  const size_t smem = horner_smem(us, sizeof(T) == 4, NU);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, W * 32, smem, st>>>(reinterpret_cast<const typename hdev::HTr<T>::V*>(Tab), S, U, us, ops, chunk, croots,
                                nchunk, out, part, full, parts, tail);
  return cudaGetLastError();
}

cudaError_t launch_horner(int nu, bool f32, const void* Tab, int64_t S, int U, int us, const OpH* ops,
                          const int32_t* chunk, const int32_t* croots, int nchunk, double* out, double* part,
                          int64_t full, int parts, double* tail, int grid, cudaStream_t st) {
  const int hot = std::min(U, horner_hot_rows(f32));
  const bool hyb = hot + us < U;
#define ACEDAG_H(N, T)                                                                                          \
  return hyb ? launch_nu<N, T, true>(Tab, S, U, us, ops, chunk, croots, nchunk, out, part, full, parts, tail,  \
                                     grid, st)                                                                \
             : launch_nu<N, T, false>(Tab, S, U, us, ops, chunk, croots, nchunk, out, part, full, parts, tail, \
                                      grid, st)
#ifdef ACEDAG_HORNER_FAST  // experiment builds: order 4 only (tools/mkvariant.sh)
  if (nu != 4) return cudaErrorInvalidValue;
  if (f32) { ACEDAG_H(4, float); }
  ACEDAG_H(4, double);
#else
  if (f32) {
    switch (nu) {
      case 2: ACEDAG_H(2, float);
      case 3: ACEDAG_H(3, float);
      case 4: ACEDAG_H(4, float);
      case 5: ACEDAG_H(5, float);
      case 6: ACEDAG_H(6, float);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (nu) {
    case 2: ACEDAG_H(2, double);
    case 3: ACEDAG_H(3, double);
    case 4: ACEDAG_H(4, double);
    case 5: ACEDAG_H(5, double);
    case 6: ACEDAG_H(6, double);
    default: return cudaErrorInvalidValue;
  }
#endif
#undef ACEDAG_H
}

}  // namespace acedag
