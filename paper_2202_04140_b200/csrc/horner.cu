// K2 Horner kernel: the recursive program evaluated bottom-up (see horner.h).
//
// Geometry (as k2_quad): one persistent CTA per SM, 16 warps, 128-site tiles;
// lane l carries sites l, l+32, l+64, l+96 of the tile, so every program
// record serves four products per lane.  The seeds of a tile are split by
// use count: the 32 hottest rows in tensor memory (16 columns per lane, one
// tcgen05.ld.32x32b.x16 per fetch, replicated in the four lane quadrants),
// the next `us` rows in shared memory ([row][4][32] c128, conflict-free
// LDS.128), the tail read in place from the tile-major table (L2).
//
// Per warp, the program records of a chunk stream global -> a 3-block shared
// ring (cp.async, one 512-B block per refill) whose block 0 is mirrored past
// block 2, so any 32 consecutive records from a checked position are
// readable without wrap logic; the refill check runs once per "unit" (a root
// pair, an inner record, or a deepest-level parent with its leaves), not per
// record.  The leaf loop is then: LDS.128 record, one TMEM (or four LDS.128)
// seed fetch, 8 DFMA.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <vector>

#include "horner.h"

namespace acedag {
namespace hdev {

extern __shared__ __align__(16) unsigned char h_smem[];

struct C4 {
  double2 v[4];
};

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t addr, double2 a, double2 b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(addr),
               "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)), "r"(__double2hiint(a.y)),
               "r"(__double2loint(b.x)), "r"(__double2hiint(b.x)), "r"(__double2loint(b.y)), "r"(__double2hiint(b.y)));
}

__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 r;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ double rec_c(int4 r) { return __hiloint2double(r.y, r.x); }

// ------------------------------------------------------------ program ring
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
template <bool HYB>
struct SeedsH {
  uint32_t tq;     // TMEM address of this warp's lane quadrant, column 0
  uint32_t sb;     // shared address of cold row 0 + lane * 16
  const char* gb;  // global tail row 0 of this tile + lane * 16
  // z: TMEM address of the row in this warp's lane quadrant (the program
  // copy of the quadrant carries the lane bits; the allocation base is 0)
  __device__ __forceinline__ void hot(uint32_t z, uint32_t (&t)[16]) const { tmem_ld16(z, t); }
  __device__ __forceinline__ static C4 unpack(const uint32_t (&t)[16]) {
    C4 s;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      s.v[k] = make_double2(__hiloint2double(t[4 * k + 1], t[4 * k]), __hiloint2double(t[4 * k + 3], t[4 * k + 2]));
    return s;
  }
  __device__ __forceinline__ C4 sm(uint32_t z) const {
    C4 s;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(s.v[k].x), "=d"(s.v[k].y) : "r"(sb + z + k * 512));
    return s;
  }
  __device__ __forceinline__ C4 gl(uint32_t z) const {
    C4 s;
#pragma unroll
    for (int k = 0; k < 4; ++k) s.v[k] = __ldg(reinterpret_cast<const double2*>(gb + z + k * 512));
    return s;
  }
  __device__ __forceinline__ C4 get(uint32_t z, uint32_t cls) const {
    if (cls == 0) {
      uint32_t t[16];
      hot(z, t);
      tmem_wait_ld();
      return unpack(t);
    }
    if (!HYB || cls == 1) return sm(z);
    return gl(z);
  }
};

__device__ __forceinline__ void init_h(C4& H, double c) {
#pragma unroll
  for (int k = 0; k < 4; ++k) H.v[k] = make_double2(c, 0.0);
}
// H += c s
__device__ __forceinline__ void axpy(C4& H, double c, const C4& s) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    H.v[k].x = __fma_rn(c, s.v[k].x, H.v[k].x);
    H.v[k].y = __fma_rn(c, s.v[k].y, H.v[k].y);
  }
}
// Hp += s H
__device__ __forceinline__ void cmac(C4& Hp, const C4& s, const C4& H) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Hp.v[k].x = __fma_rn(s.v[k].x, H.v[k].x, Hp.v[k].x);
    Hp.v[k].y = __fma_rn(s.v[k].x, H.v[k].y, Hp.v[k].y);
    Hp.v[k].x = __fma_rn(-s.v[k].y, H.v[k].y, Hp.v[k].x);
    Hp.v[k].y = __fma_rn(s.v[k].y, H.v[k].x, Hp.v[k].y);
  }
}

__device__ __forceinline__ uint32_t w_nch(uint32_t w) { return w & 0xFFFFu; }
__device__ __forceinline__ uint32_t w_nhot(uint32_t w) { return (w >> 16) & 63u; }
__device__ __forceinline__ uint32_t w_nsm(uint32_t w) { return w >> 22; }

// ---------------------------------------------------------------- program walk
template <uint32_t PC, bool HYB>
__device__ __forceinline__ C4 seed_of(const SeedsH<HYB>& sd, uint32_t z) {
  if constexpr (PC == 0) {
    uint32_t t[16];
    sd.hot(z, t);
    tmem_wait_ld();
    return SeedsH<HYB>::unpack(t);
  } else if constexpr (PC == 1) {
    return sd.sm(z);
  } else {
    return sd.gl(z);
  }
}

// H = c + c_l s (the accumulator's first term folded into its FMAs)
__device__ __forceinline__ void axpy_init(C4& H, double c, double cl, const C4& s) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    H.v[k].x = __fma_rn(cl, s.v[k].x, c);
    H.v[k].y = __dmul_rn(cl, s.v[k].y);
  }
}

// hot leaves [q, qh) two per TMEM round trip
template <bool HYB>
__device__ __forceinline__ void hot_leaves(uint32_t q, uint32_t qh, C4& H, const SeedsH<HYB>& sd) {
#pragma unroll 1
  for (; q + 16 < qh; q += 32) {
    const int4 r0 = lds128(q), r1 = lds128(q + 16);
    uint32_t t0[16], t1[16];
    sd.hot((uint32_t)r0.z, t0);
    sd.hot((uint32_t)r1.z, t1);
    tmem_wait_ld();
    axpy(H, rec_c(r0), SeedsH<HYB>::unpack(t0));
    axpy(H, rec_c(r1), SeedsH<HYB>::unpack(t1));
  }
  if (q < qh) {
    const int4 r = lds128(q);
    axpy(H, rec_c(r), seed_of<0, HYB>(sd, (uint32_t)r.z));
  }
}

// H = c + sum over the leaves (maximum order) of one node, whose records
// start at q (first: l, already read): hot, shared, global -- at most
// kMaxLeaves, so they lie in the checked ring window.  The first leaf's FMA
// carries c; a node whose leaves are all hot (the usual case) skips the
// other loops.
template <bool HYB>
__device__ __forceinline__ void leaves(uint32_t q, uint32_t w, double c, int4 l, C4& H, const SeedsH<HYB>& sd) {
  const uint32_t nh = w_nhot(w), ns = w_nsm(w), n = w_nch(w);
  const uint32_t qh = q + nh * 16, qs = qh + ns * 16, qe = q + n * 16;
  if (nh) {
    axpy_init(H, c, rec_c(l), seed_of<0, HYB>(sd, (uint32_t)l.z));
    hot_leaves<HYB>(q + 16, qh, H, sd);
    if (nh == n) return;
    q = qh;
  } else if (n) {
    axpy_init(H, c, rec_c(l), ns ? sd.sm((uint32_t)l.z) : sd.gl((uint32_t)l.z));
    q += 16;
  } else {
    init_h(H, c);
    return;
  }
#pragma unroll 1
  for (; q < qs; q += 16) {
    const int4 r = lds128(q);
    axpy(H, rec_c(r), sd.sm((uint32_t)r.z));
  }
  if constexpr (HYB) {
#pragma unroll 1
    for (; q < qe; q += 16) {
      const int4 r = lds128(q);
      axpy(H, rec_c(r), sd.gl((uint32_t)r.z));
    }
  }
}

// n sibling nodes of order NU-1 whose seeds are of class PC; each adds
// s * (c + sum_leaves c_l s_l) to Hp.  The node record and the one after it
// (its first leaf) are read together; for the commonest shape (one hot
// leaf) the leaf seed and a hot node seed are fetched by one TMEM round trip.
template <uint32_t PC, bool HYB>
__device__ __forceinline__ void parents(RingH& st, uint32_t n, C4& Hp, const SeedsH<HYB>& sd, int lane) {
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const int4 r = st.at(0), l = st.at(1);
    const uint32_t w = (uint32_t)r.w;
    C4 H, sp;
    if (w == (1u | 1u << 16)) {  // one hot leaf (the commonest shape)
      uint32_t tl[16];
      sd.hot((uint32_t)l.z, tl);
      if constexpr (PC == 0) {
        uint32_t tp[16];
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SeedsH<HYB>::unpack(tp);
      } else {
        tmem_wait_ld();
      }
      axpy_init(H, rec_c(r), rec_c(l), SeedsH<HYB>::unpack(tl));
    } else if (w == (2u | 2u << 16)) {  // two hot leaves (the next commonest)
      const int4 l2 = st.at(2);
      uint32_t tl[16], tl2[16];
      sd.hot((uint32_t)l.z, tl);
      sd.hot((uint32_t)l2.z, tl2);
      if constexpr (PC == 0) {
        uint32_t tp[16];
        sd.hot((uint32_t)r.z, tp);
        tmem_wait_ld();
        sp = SeedsH<HYB>::unpack(tp);
      } else {
        tmem_wait_ld();
      }
      axpy_init(H, rec_c(r), rec_c(l), SeedsH<HYB>::unpack(tl));
      axpy(H, rec_c(l2), SeedsH<HYB>::unpack(tl2));
    } else {
      leaves<HYB>(st.p + 16, w, rec_c(r), l, H, sd);
      if constexpr (PC == 0) sp = seed_of<0, HYB>(sd, (uint32_t)r.z);
    }
    if constexpr (PC != 0) sp = seed_of<PC, HYB>(sd, (uint32_t)r.z);
    cmac(Hp, sp, H);
    st.p += 16 * (1 + w_nch(w));
    st.check(lane);
  }
}

template <int D, int NU, bool HYB>
__device__ __forceinline__ void children(RingH& st, uint32_t w, C4& Hp, const SeedsH<HYB>& sd, int lane);

// n sibling nodes of order D < NU-1 with seeds of class PC
template <int D, int NU, uint32_t PC, bool HYB>
__device__ __forceinline__ void inner(RingH& st, uint32_t n, C4& Hp, const SeedsH<HYB>& sd, int lane) {
#pragma unroll 1
  for (uint32_t j = 0; j < n; ++j) {
    const int4 r = st.at(0);
    st.p += 16;
    st.check(lane);
    C4 H;
    init_h(H, rec_c(r));
    children<D + 1, NU, HYB>(st, (uint32_t)r.w, H, sd, lane);
    cmac(Hp, seed_of<PC, HYB>(sd, (uint32_t)r.z), H);
  }
}

// the children (order D) of a node whose accumulator is Hp, by seed class;
// the ring was checked right before the first child record
template <int D, int NU, bool HYB>
__device__ __forceinline__ void children(RingH& st, uint32_t w, C4& Hp, const SeedsH<HYB>& sd, int lane) {
  const uint32_t nh = w_nhot(w), ns = w_nsm(w), ng = w_nch(w) - nh - ns;
  if constexpr (D == NU - 1) {
    parents<0, HYB>(st, nh, Hp, sd, lane);
    parents<1, HYB>(st, ns, Hp, sd, lane);
    if (HYB) parents<2, HYB>(st, ng, Hp, sd, lane);
  } else if constexpr (D < NU - 1) {
    inner<D, NU, 0, HYB>(st, nh, Hp, sd, lane);
    inner<D, NU, 1, HYB>(st, ns, Hp, sd, lane);
    if (HYB) inner<D, NU, 2, HYB>(st, ng, Hp, sd, lane);
  }
}

template <int NU, bool HYB>
__device__ __forceinline__ void root(RingH& st, double (&acc)[4], const SeedsH<HYB>& sd, int lane) {
  const int4 r0 = st.at(0), r1 = st.at(1);
  const double c = rec_c(r0);
  const uint32_t fl = (uint32_t)r1.w;
  C4 H;
  if constexpr (NU == 3) {
    leaves<HYB>(st.p + 32, (uint32_t)r0.w, c, st.at(2), H, sd);
    st.p += 16 * (2 + w_nch((uint32_t)r0.w));
    st.check(lane);
  } else {
    init_h(H, c);
    st.p += 32;
    st.check(lane);
    if constexpr (NU >= 4) children<3, NU, HYB>(st, (uint32_t)r0.w, H, sd, lane);
  }
  const C4 sa = sd.get((uint32_t)r0.z, fl & 3u);
  if (fl & 16u) {  // order-1 coefficient: c Re(s_a)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = __fma_rn(c, sa.v[k].x, acc[k]);
  } else {
    const C4 sb = sd.get((uint32_t)r1.z, (fl >> 2) & 3u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double abx = __fma_rn(sa.v[k].x, sb.v[k].x, -__dmul_rn(sa.v[k].y, sb.v[k].y));
      const double aby = __fma_rn(sa.v[k].x, sb.v[k].y, __dmul_rn(sa.v[k].y, sb.v[k].x));
      acc[k] = __fma_rn(abx, H.v[k].x, acc[k]);
      acc[k] = __fma_rn(-aby, H.v[k].y, acc[k]);
    }
  }
}

// T: tile-major seed table [ntiles][U + 1][128] c128
template <int NU, bool HYB, int W>
__global__ void __launch_bounds__(W * 32, 1)
k2_horner(const double2* __restrict__ T, int64_t S, int U, int us, const OpH* __restrict__ ops,
          const int32_t* __restrict__ chunk, const int32_t* __restrict__ croots, int nchunk,
          double* __restrict__ out, double* __restrict__ part, int64_t full_tiles, int tail_parts,
          double* __restrict__ tailbuf) {
  unsigned char* smem = h_smem;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = U + 1;  // table rows (row U: the constant ONE, unused here)
  const int hot = U < (int)kHornerHot ? U : (int)kHornerHot;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t rings = sbase + (uint32_t)us * 2048u;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + (size_t)us * 2048 + W * kHornerRing);
  int* dyn = reinterpret_cast<int*>(tslot) + 1;
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
  SeedsH<HYB> sd;
  sd.tq = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  sd.sb = sbase + (uint32_t)(lane * 16);
  sd.gb = nullptr;
  const uint32_t ring = rings + (uint32_t)warp * kHornerRing;
  const int32_t nops = __ldg(chunk + nchunk);  // records per quadrant copy
  double* mypart = part + (size_t)blockIdx.x * nchunk * 128;
  RingH st;
  const int64_t ntiles = (S + 127) / 128;
  const int64_t nitems = full_tiles + (ntiles - full_tiles) * tail_parts;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const bool whole = it < full_tiles;
    const int64_t tile = whole ? it : full_tiles + (it - full_tiles) / tail_parts;
    const int slice = whole ? 0 : (int)((it - full_tiles) % tail_parts);
    const int nsl = whole ? 1 : tail_parts;
    const int cb = (int)((int64_t)slice * nchunk / nsl), ce = (int)((int64_t)(slice + 1) * nchunk / nsl);
    const double2* Tt = T + tile * (int64_t)rows * 128;
    // the next item's on-chip rows into L2 while this tile computes
    if (threadIdx.x == 0 && it + gridDim.x < nitems) {
      const int64_t nit = it + gridDim.x;
      const int64_t nt = nit < full_tiles ? nit : full_tiles + (nit - full_tiles) / tail_parts;
      if (nt != tile) {
        const char* src = reinterpret_cast<const char*>(T + nt * (int64_t)rows * 128);
        const uint32_t bytes = (uint32_t)(hot + us) * 2048u;
        for (uint32_t o = 0; o < bytes; o += 32768u) {
          const uint32_t n = bytes - o < 32768u ? bytes - o : 32768u;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src + o), "r"(n) : "memory");
        }
      }
    }
    if (HYB) sd.gb = reinterpret_cast<const char*>(Tt + (size_t)(hot + us) * 128) + lane * 16;
    // TMEM rows: each lane quadrant's four warps write all hot rows
    for (int h0 = warp >> 2; h0 < hot; h0 += 4 * (W / 4)) {
      double2 v[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (W / 4);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          v[q][k] = h < hot ? ld_stream(Tt + (size_t)h * 128 + k * 32 + lane) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int h = h0 + q * (W / 4);
        if (h < hot) {
          tmem_st8(sd.tq + (uint32_t)h * 16, v[q][0], v[q][1]);
          tmem_st8(sd.tq + (uint32_t)h * 16 + 8, v[q][2], v[q][3]);
        }
      }
    }
    // shared rows: asynchronous 16-byte copies
    for (int idx = threadIdx.x; idx < us * 128; idx += W * 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + idx * 16),
                   "l"(Tt + (size_t)hot * 128 + idx)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (threadIdx.x == 0) *dyn = cb + W;
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    double* dst = whole ? mypart : tailbuf + (size_t)((it - full_tiles) / tail_parts) * nchunk * 128;
    for (int ci = cb + warp; ci < ce;) {
      const int32_t b = __ldg(chunk + ci), e = __ldg(chunk + ci + 1);
      const int32_t nr = __ldg(croots + ci);
      st.begin(reinterpret_cast<const int4*>(ops) + (size_t)(warp & 3) * nops + b, (uint32_t)(e - b), ring, lane);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int32_t k = 0; k < nr; ++k) root<NU, HYB>(st, acc, sd, lane);
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

}  // namespace hdev

// ------------------------------------------------------------------- host
// warps per CTA (ACEDAG_HWARPS = 16 | 20 | 24)
int horner_warps() {
  static int w = [] {
    const char* e = getenv("ACEDAG_HWARPS");
    const int v = e ? atoi(e) : kHornerWarps;
    return v == 20 || v == 24 ? v : 16;
  }();
  return w;
}

int horner_us_max(size_t smem_optin) {
  const size_t fixed = (size_t)horner_warps() * kHornerRing + 16;
  return smem_optin > fixed ? (int)((smem_optin - fixed) / 2048) : 0;
}
size_t horner_smem(int us) { return (size_t)us * 2048 + (size_t)horner_warps() * kHornerRing + 16; }

namespace {
uint32_t w_count(uint32_t w) { return w & 0xFFFFu; }
// relative size of the second half of the chunks (ACEDAG_HGUIDE; 1 = equal)
double guided_tail() {
  static double v = [] {
    const char* e = getenv("ACEDAG_HGUIDE");
    const double x = e ? atof(e) : 1.0;
    return x > 0 ? x : 1.0;
  }();
  return v;
}
struct HornerEnc {
  const PlanHost& H;
  uint32_t hot, us, U;
  int nu;
  std::vector<OpH>& out;
  std::vector<uint8_t> hot_rec;  // record's z is a TMEM column (gets the lane-quadrant bits per copy)
  bool ok = true;

  uint32_t cls(uint32_t s) const { return s < hot ? 0u : (s < hot + us ? 1u : 2u); }
  uint32_t zof(uint32_t s) const {
    const uint32_t c = cls(s);
    return c == 0 ? s * 16u : (c == 1 ? (s - hot) * 2048u : (s - hot - us) * 2048u);
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
    if (n > 0xFFFFu || nh > 63u || ns > 1023u) ok = false;
    return n | nh << 16 | ns << 22;
  }
  // leaves [first, first + n) of a node (positions of records with nch = 0)
  void emit_leaves(const std::vector<size_t>& kids, size_t b, size_t e) {
    for (size_t j = b; j < e; ++j) {
      const Op& l = H.ops[kids[j]];
      out.push_back(OpH{l.c, zof(slot(l)), 0u});
      hot_rec.push_back(cls(slot(l)) == 0);
    }
  }
  uint32_t leaf_w(const std::vector<size_t>& kids, size_t b, size_t e) {
    uint32_t n = 0, nh = 0, ns = 0;
    for (size_t j = b; j < e; ++j) count(cls(slot(H.ops[kids[j]])), 1, n, nh, ns);
    return pack(n, nh, ns);
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
    const uint8_t zh = cls(slot(o)) == 0;
    if (d == nu) {
      out.push_back(OpH{o.c, z, 0u});
      hot_rec.push_back(zh);
      return 1;
    }
    if (d == nu - 1) {
      uint32_t copies = 0;
      size_t b = 0;
      do {
        const size_t e = std::min(kids.size(), b + kMaxLeaves);
        out.push_back(OpH{b == 0 ? o.c : 0.0, z, leaf_w(kids, b, e)});
        hot_rec.push_back(zh);
        emit_leaves(kids, b, e);
        copies++;
        b = e;
      } while (b < kids.size());
      return copies;
    }
    const size_t me = out.size();
    out.push_back(OpH{o.c, z, 0u});
    hot_rec.push_back(zh);
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
    const std::vector<size_t> kids = kids_from(pos + 2, a.nch);  // children follow the pair
    if (nu == 3) {
      size_t bb = 0;
      bool first = true;
      do {
        const size_t e = std::min(kids.size(), bb + kMaxLeaves);
        out.push_back(OpH{first ? a.c : 0.0, zof(sa), leaf_w(kids, bb, e)});
        out.push_back(OpH{0.0, single ? 0u : zof(sb), fl});
        hot_rec.push_back(cls(sa) == 0);
        hot_rec.push_back(!single && cls(sb) == 0);
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
      uint32_t n = 0, nh = 0, ns = 0;
      for (size_t k : kids) count(cls(slot(H.ops[k])), node(k, 3), n, nh, ns);
      out[me].w = pack(n, nh, ns);
      nroots++;
    }
    size_t q = pos + 2;
    for (size_t j = 0; j < kids.size(); ++j) q = skip(q);
    return q;
  }
  int32_t nroots = 0;
};
}  // namespace

bool encode_horner(const PlanHost& H, uint32_t hot, uint32_t us, std::vector<OpH>& out,
                   std::vector<int32_t>& chunk, std::vector<int32_t>& croots) {
  out.clear();
  const size_t nchunk = H.chunk.size() > 0 ? H.chunk.size() - 1 : 0;
  HornerEnc E{H, hot, us, (uint32_t)H.slot_label.size(), H.max_order, out};
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
        const size_t e = E.nroots - r0 == 1 ? out.size() : q + 2 + w_count(out[q].w);
        start.push_back(q);
        double c = 2.0;
        for (size_t t = q; t < e; ++t) c += (t != q + 1 && out[t].w) ? 3.0 : 1.0;
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
  out.resize(4 * n);
  for (size_t q = 1; q < 4; ++q)
    for (size_t i = 0; i < n; ++i) {
      out[q * n + i] = out[i];
      if (E.hot_rec[i]) out[q * n + i].z += (uint32_t)(q * 32) << 16;
    }
  return E.ok && 4 * n < (size_t)INT32_MAX;
}

template <int NU, bool HYB>
static cudaError_t launch_nu(const double2* T, int64_t S, int U, int us, const OpH* ops, const int32_t* chunk,
                             const int32_t* croots, int nchunk, double* out, double* part, int64_t full, int parts,
                             double* tail, int grid, cudaStream_t st) {
  const int W = horner_warps();
  auto k = W == 24 ? hdev::k2_horner<NU, HYB, 24> : (W == 20 ? hdev::k2_horner<NU, HYB, 20> : hdev::k2_horner<NU, HYB, 16>);
  const size_t smem = horner_smem(us);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, W * 32, smem, st>>>(T, S, U, us, ops, chunk, croots, nchunk, out, part, full, parts, tail);
  return cudaGetLastError();
}

cudaError_t launch_horner(int nu, const double2* T, int64_t S, int U, int us, const OpH* ops,
                          const int32_t* chunk, const int32_t* croots, int nchunk, double* out, double* part,
                          int64_t full, int parts, double* tail, int grid, cudaStream_t st) {
  const int hot = std::min(U, (int)kHornerHot);
  const bool hyb = hot + us < U;
#define ACEDAG_H(N)                                                                                          \
  return hyb ? launch_nu<N, true>(T, S, U, us, ops, chunk, croots, nchunk, out, part, full, parts, tail, grid, \
                                  st)                                                                        \
             : launch_nu<N, false>(T, S, U, us, ops, chunk, croots, nchunk, out, part, full, parts, tail, grid, st)
  switch (nu) {
    case 2: ACEDAG_H(2);
    case 3: ACEDAG_H(3);
    case 4: ACEDAG_H(4);
    case 5: ACEDAG_H(5);
    case 6: ACEDAG_H(6);
    default: return cudaErrorInvalidValue;
  }
#undef ACEDAG_H
}

}  // namespace acedag
