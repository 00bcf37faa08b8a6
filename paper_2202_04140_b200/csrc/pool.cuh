// K1: the atomic basis (pool).
//
// pool_ref<GROUP>: the reference convention (evaluator.py:61-90) for all four
// groups, one thread per (site, label), particles summed in order from 0j.
// Recurrences use explicit round-to-nearest intrinsics so the compiler does
// not contract them into FMAs: chebyshev (special.py:19-28), the upward-l
// associated Legendre recursion with Condon-Shortley phase (special.py:31-47)
// and the exact-factorial norm table (special.py:57-59, ylm_norms.h).  Only
// cos/sin may differ from the host libm by an ulp.
//
// pool_positions: BASELINE cfg3/cfg5 -- Cartesian neighbour vectors, one CTA
// per site: per-neighbour radial/Legendre/phase tables are built once in
// shared memory, then every label is a J-term dot product.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ylm_norms.h"

namespace acedag {
namespace dev {

__constant__ double c_ylm_norm[(ACEDAG_YLM_LMAX + 1) * (ACEDAG_YLM_LMAX + 2) / 2];
__constant__ double c_recip[ACEDAG_YLM_LMAX + 2];  // 1/k, k = 0..LMAX+1 (entry 0 unused)
// recurrence of the normalised Q_l^m = N_lm P_l^m (capi.cu ensure_norms):
// Q_l^m = c_ylm_a[l,m] cos(theta) Q_{l-1}^m - c_ylm_b[l,m] Q_{l-2}^m
__constant__ double c_ylm_a[(ACEDAG_YLM_LMAX + 1) * (ACEDAG_YLM_LMAX + 2) / 2];
__constant__ double c_ylm_b[(ACEDAG_YLM_LMAX + 1) * (ACEDAG_YLM_LMAX + 2) / 2];

__device__ __forceinline__ double cheb_exact(int k, double x) {  // special.py:19-28
  if (k == 0) return 1.0;
  double prev = 1.0, cur = x;
  const double two_x = __dmul_rn(2.0, x);
  for (int i = 0; i < k - 1; ++i) {
    double nxt = __dsub_rn(__dmul_rn(two_x, cur), prev);
    prev = cur;
    cur = nxt;
  }
  return cur;
}

__device__ __forceinline__ double legendre_exact(int l, int m, double x) {  // special.py:31-47
  const double sx = __dsqrt_rn(fmax(0.0, __dmul_rn(__dsub_rn(1.0, x), __dadd_rn(1.0, x))));
  double pmm = 1.0;
  for (int k = 1; k <= m; ++k) pmm = __dmul_rn(pmm, __dmul_rn((double)(-(2 * k - 1)), sx));
  if (l == m) return pmm;
  double pm1 = __dmul_rn(__dmul_rn(x, (double)(2 * m + 1)), pmm);
  if (l == m + 1) return pm1;
  for (int ll = m + 2; ll <= l; ++ll) {
    double t = __dsub_rn(__dmul_rn(__dmul_rn(x, (double)(2 * ll - 1)), pm1),
                         __dmul_rn((double)(ll + m - 1), pmm));
    pmm = pm1;
    pm1 = __ddiv_rn(t, (double)(ll - m));
  }
  return pm1;
}

// Y_l^m(theta, phi) as the reference computes it (special.py:50-63)
__device__ __forceinline__ double2 sph_harm_exact(int l, int m, double theta, double phi) {
  const int am = m < 0 ? -m : m;
  const double np = __dmul_rn(c_ylm_norm[l * (l + 1) / 2 + am], legendre_exact(l, am, cos(theta)));
  double sn, cs;
  sincos(__dmul_rn((double)am, phi), &sn, &cs);
  double2 y = make_double2(__dmul_rn(np, cs), __dmul_rn(np, sn));
  if (m < 0) {
    const double sg = (am & 1) ? -1.0 : 1.0;
    y = make_double2(__dmul_rn(sg, y.x), -__dmul_rn(sg, y.y));
  }
  return y;
}

// labels: int4 (n, l, m, f) per label, or (m,0,0,0) for T and (n,m,0,0) for SO2
template <int GROUP>
__global__ void pool_ref(const double* __restrict__ coords, const int32_t* __restrict__ counts,
                         int64_t S, int J, const int4* __restrict__ labels, int L,
                         double2* __restrict__ out) {
  constexpr int NC = GROUP == 0 ? 1 : (GROUP == 1 ? 2 : (GROUP == 2 ? 3 : 4));
  const int64_t total = S * (int64_t)L;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = idx / L;
    const int4 e = labels[idx - s * L];
    const int nj = counts ? min(max(counts[s], 0), J) : J;  // ragged sites, clamped to the row
    double ar = 0.0, ai = 0.0;
    for (int j = 0; j < nj; ++j) {
      const double* c = coords + (s * J + j) * NC;
      double vr, vi;
      if (GROUP == 0) {  // e^{i m theta}
        double sn, cs;
        sincos(__dmul_rn((double)e.x, c[0]), &sn, &cs);
        vr = cs;
        vi = sn;
      } else if (GROUP == 1) {  // R_n(r) e^{-i m theta}
        const double R = cheb_exact(e.x, __dsub_rn(__dmul_rn(2.0, c[0]), 1.0));
        double sn, cs;
        sincos(__dmul_rn((double)(-e.y), c[1]), &sn, &cs);
        vr = __dmul_rn(R, cs);
        vi = __dmul_rn(R, sn);
      } else {  // R_n(r) Y_l^m [T_f(mu)]
        const double R = cheb_exact(e.x, __dsub_rn(__dmul_rn(2.0, c[0]), 1.0));
        const double2 y = sph_harm_exact(e.y, e.z, c[1], c[2]);
        vr = __dmul_rn(R, y.x);
        vi = __dmul_rn(R, y.y);
        if (GROUP == 3) {
          const double tf = cheb_exact(e.w, c[3]);
          vr = __dmul_rn(vr, tf);
          vi = __dmul_rn(vi, tf);
        }
      }
      ar = __dadd_rn(ar, vr);
      ai = __dadd_rn(ai, vi);
    }
    out[idx] = make_double2(ar, ai);
  }
}

// ------------------------------------------------------------ positions
// Per-neighbour table layout in smem (doubles): w | R[0..cap] | cos m phi,
// sin m phi [0..cap] | Pbar[l(l+1)/2 + m] for l <= cap.
__host__ __device__ inline int pos_stride(int cap) {
  return 1 + (cap + 1) + 2 * (cap + 1) + (cap + 1) * (cap + 2) / 2;
}

__global__ void pool_positions(const double* __restrict__ xyz, const int32_t* __restrict__ counts,
                               int64_t S, int J, int cap, double r_in, double r_cut,
                               const int4* __restrict__ labels, int L,
                               const int32_t* __restrict__ out_labels, int L_out, int64_t out_stride,
                               double2* __restrict__ out) {
  extern __shared__ double tabs[];
  const int st = pos_stride(cap);
  const double inv_span = 1.0 / (r_cut - r_in);
  for (int64_t s = blockIdx.x; s < S; s += gridDim.x) {
    const int nj = counts ? min(counts[s], J) : J;
    for (int j = threadIdx.x; j < nj; j += blockDim.x) {
      double* t = tabs + j * st;
      const double* p = xyz + (s * J + j) * 3;
      const double x = p[0], y = p[1], z = p[2];
      const double rho2 = x * x + y * y;
      const double r = sqrt(rho2 + z * z);
      const double w = r < r_cut ? 0.5 * (1.0 + cospi(r / r_cut)) : 0.0;
      t[0] = w;
      // radial: T_n(2 xs - 1), xs = (r - r_in)/(r_cut - r_in) clamped
      const double xs = fmin(1.0, fmax(0.0, (r - r_in) * inv_span));
      const double u = 2.0 * xs - 1.0;
      double* R = t + 1;
      R[0] = 1.0;
      if (cap >= 1) R[1] = u;
      for (int n = 2; n <= cap; ++n) R[n] = 2.0 * u * R[n - 1] - R[n - 2];
      // azimuthal phase e^{i m phi} by complex powers of (x + i y)/rho
      double* E = R + (cap + 1);
      const double rho = sqrt(rho2);
      double ec = 1.0, es = 0.0;
      if (rho > 0.0) { ec = x / rho; es = y / rho; }
      double pc = 1.0, ps = 0.0;
      for (int m = 0; m <= cap; ++m) {
        E[2 * m] = pc;
        E[2 * m + 1] = ps;
        const double nc = pc * ec - ps * es;
        ps = pc * es + ps * ec;
        pc = nc;
      }
      // normalised associated Legendre, ct = cos theta, stt = sin theta
      double* Pb = E + 2 * (cap + 1);
      const double ct = r > 0.0 ? z / r : 1.0;
      const double stt = r > 0.0 ? rho / r : 0.0;
      double pmm = 1.0;
      for (int m = 0; m <= cap; ++m) {
        if (m > 0) pmm *= -(2.0 * m - 1.0) * stt;
        double p0 = pmm;
        Pb[m * (m + 1) / 2 + m] = c_ylm_norm[m * (m + 1) / 2 + m] * p0;
        if (m + 1 <= cap) {
          double p1 = ct * (2.0 * m + 1.0) * p0;
          Pb[(m + 1) * (m + 2) / 2 + m] = c_ylm_norm[(m + 1) * (m + 2) / 2 + m] * p1;
          for (int l = m + 2; l <= cap; ++l) {
            const double p2 = (ct * (2.0 * l - 1.0) * p1 - (l + m - 1.0) * p0) / (double)(l - m);
            Pb[l * (l + 1) / 2 + m] = c_ylm_norm[l * (l + 1) / 2 + m] * p2;
            p0 = p1;
            p1 = p2;
          }
        }
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L_out; k += blockDim.x) {
      const int lab = out_labels ? out_labels[k] : k;
      const int4 e = labels[lab];  // (n, l, m, 0)
      const int am = e.z < 0 ? -e.z : e.z;
      const int pidx = 1 + (cap + 1) + 2 * (cap + 1) + e.y * (e.y + 1) / 2 + am;
      double ar = 0.0, ai = 0.0;
      for (int j = 0; j < nj; ++j) {
        const double* t = tabs + j * st;
        const double a = t[0] * t[1 + e.x] * t[pidx];
        ar += a * t[1 + (cap + 1) + 2 * am];
        ai += a * t[1 + (cap + 1) + 2 * am + 1];
      }
      if (e.z < 0) {  // Y_l^{-m} = (-1)^m conj(Y_l^m)
        const double sg = (am & 1) ? -1.0 : 1.0;
        ar = sg * ar;
        ai = -sg * ai;
      }
      out[s * out_stride + k] = make_double2(ar, ai);
    }
    __syncthreads();
  }
}

}  // namespace dev
}  // namespace acedag

namespace acedag {
namespace dev {

// ------------------------------------------------------- positions, v2
// One CTA per site (grid-stride).  Phase A: per neighbour the weighted radial
// row WR[j][n] = f_c(r_j) T_n(2x_j - 1) and the direction (cos t, sin t,
// e^{i phi}).  Phase B: per (neighbour, m) the normalised Legendre column and
// Y[j][l(l+1)/2 + m] = Nbar_lm P_l^m e^{i m phi} for m >= 0.  Phase C: one
// thread per (l, m >= 0) accumulates A[n, l, m] = sum_j WR[j][n] Y[j][lm] for
// Phase C: one thread per (n, l, m >= 0) triple (tri table, only the triples
// some output needs) accumulates A[n, l, m] = sum_j WR[j][n] Y[j][lm];
// A[n, l, -m] = (-1)^m conj(A[n, l, m]) (real weights), so only half of the
// labels are computed.  col_of maps a label to its output column (-1: not
// needed); NULL writes every label at its own index.
__global__ void __launch_bounds__(256)
pool_positions2(const double* __restrict__ xyz, const int32_t* __restrict__ counts, int64_t S, int J,
                int cap, double r_in, double r_cut, const int4* __restrict__ tri, int ntri,
                const int32_t* __restrict__ col_of, int64_t out_stride, double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char psm[];
  const int npair = (cap + 1) * (cap + 2) / 2;
  double2* Y = reinterpret_cast<double2*>(psm);                  // [J][npair]
  double* WR = reinterpret_cast<double*>(Y + (size_t)J * npair);   // [J][cap+1]
  double* G = WR + (size_t)J * (cap + 1);                         // [J][4]
  const double inv_span = 1.0 / (r_cut - r_in);
  for (int64_t s = blockIdx.x; s < S; s += gridDim.x) {
    const int nj = counts ? min(counts[s], J) : J;
    for (int j = threadIdx.x; j < nj; j += blockDim.x) {
      const double* p = xyz + (s * J + j) * 3;
      const double x = p[0], y = p[1], z = p[2];
      const double rho2 = x * x + y * y;
      const double r = sqrt(rho2 + z * z);
      const double w = r < r_cut ? 0.5 * (1.0 + cospi(r / r_cut)) : 0.0;
      const double u = 2.0 * fmin(1.0, fmax(0.0, (r - r_in) * inv_span)) - 1.0;
      double* wr = WR + j * (cap + 1);
      double t0 = 1.0, t1 = u;
      wr[0] = w;
      if (cap >= 1) wr[1] = w * u;
      for (int n = 2; n <= cap; ++n) {
        const double t2 = 2.0 * u * t1 - t0;
        wr[n] = w * t2;
        t0 = t1;
        t1 = t2;
      }
      const double rho = sqrt(rho2);
      G[4 * j + 0] = r > 0.0 ? z / r : 1.0;     // cos theta
      G[4 * j + 1] = r > 0.0 ? rho / r : 0.0;   // sin theta
      G[4 * j + 2] = rho > 0.0 ? x / rho : 1.0; // cos phi
      G[4 * j + 3] = rho > 0.0 ? y / rho : 0.0; // sin phi
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nj * (cap + 1); idx += blockDim.x) {
      const int j = idx / (cap + 1), m = idx - j * (cap + 1);
      const double4 g = make_double4(G[4 * j], G[4 * j + 1], G[4 * j + 2], G[4 * j + 3]);
      double ec = 1.0, es = 0.0;  // e^{i m phi}
      for (int k = 0; k < m; ++k) {
        const double nc = ec * g.z - es * g.w;
        es = ec * g.w + es * g.z;
        ec = nc;
      }
      double pmm = 1.0;
      for (int k = 1; k <= m; ++k) pmm *= -(2.0 * k - 1.0) * g.y;
      double2* yj = Y + (size_t)j * npair;
      double nv = c_ylm_norm[m * (m + 1) / 2 + m] * pmm;
      yj[m * (m + 1) / 2 + m] = make_double2(nv * ec, nv * es);
      if (m + 1 <= cap) {
        double p0 = pmm, p1 = g.x * (2.0 * m + 1.0) * pmm;
        nv = c_ylm_norm[(m + 1) * (m + 2) / 2 + m] * p1;
        yj[(m + 1) * (m + 2) / 2 + m] = make_double2(nv * ec, nv * es);
        for (int l = m + 2; l <= cap; ++l) {
          const double p2 = (g.x * (2.0 * l - 1.0) * p1 - (l + m - 1.0) * p0) * c_recip[l - m];
          nv = c_ylm_norm[l * (l + 1) / 2 + m] * p2;
          yj[l * (l + 1) / 2 + m] = make_double2(nv * ec, nv * es);
          p0 = p1;
          p1 = p2;
        }
      }
    }
    __syncthreads();
    // phase C: one thread per (n, l, m >= 0) triple of the table
    for (int t = threadIdx.x; t < ntri; t += blockDim.x) {
      const int4 q = __ldg(tri + t);  // (n, l, m, label index of (n, l, m))
      const int pair = q.y * (q.y + 1) / 2 + q.z;
      double ar = 0.0, ai = 0.0;
      for (int j = 0; j < nj; ++j) {
        const double2 yv = Y[(size_t)j * npair + pair];
        const double a = WR[j * (cap + 1) + q.x];
        ar += a * yv.x;
        ai += a * yv.y;
      }
      const int cp = col_of ? col_of[q.w] : q.w;
      if (cp >= 0) out[s * out_stride + cp] = make_double2(ar, ai);
      if (q.z > 0) {  // A[n, l, -m] = (-1)^m conj(A[n, l, m])
        const int lab_m = q.w - 2 * q.z;
        const int cm = col_of ? col_of[lab_m] : lab_m;
        const double sg = (q.z & 1) ? -1.0 : 1.0;
        if (cm >= 0) out[s * out_stride + cm] = make_double2(sg * ar, -sg * ai);
      }
    }
    __syncthreads();
  }
}

inline size_t pool2_smem(int cap, int J) {
  const size_t npair = (size_t)(cap + 1) * (cap + 2) / 2;
  return (size_t)J * npair * 16 + (size_t)J * (cap + 1) * 8 + (size_t)J * 32;
}

}  // namespace dev
}  // namespace acedag

namespace acedag {
namespace dev {

// ------------------------------------------------------- positions, v4
// Degree cap as a template parameter (cfg2/3: 12, cfg5: 14): one WARP per
// site, lane = neighbour.  Each lane evaluates its neighbour's weighted
// radial row and the whole Y_lm table (m outer, the upward Legendre
// recursion in l inner) as straight-line code with compile-time indices
// and constants -- no per-(j, m) work items, no divergent trip counts --
// into shared memory Y[j][pair] (row stride odd in 16-B units: conflict-free
// for both the lane = j writes and the lane = triple reads).  Then every
// lane accumulates its TPL (n, l, m >= 0) triples A = sum_j WR[j][n] Y[j][lm]
// in registers, j ascending, NB neighbours per pass.  (Round 2: splitting
// each neighbour's table over two lanes by the parity of m, so every lane
// works in the table phase, ran 2.1 vs 1.92 ms per 131k-site cfg3 chunk.)
template <int CAP, bool PRUNE = false, int NB = 16>
struct Pool4Geom {
  static constexpr int kNB = NB;  // neighbours per pass (lanes computing Y)
  static constexpr int kC1 = CAP + 1;
  // Y_lm pairs (l, m >= 0) in the table: all of them, or (PRUNE) only those
  // with l + m <= CAP, ordered by m then l.  The PRUNE row is sized for
  // (CAP/2 + 1)(CAP + 2 - CAP/2) entries (56 at cap 12, 49 used): that stride
  // measured 36.3 ms per cfg3 step against 38.6 ms for an l-major table of
  // exactly 49 entries
  static constexpr int kNP = PRUNE ? (CAP / 2 + 1) * (CAP + 2 - CAP / 2) : kC1 * (CAP + 2) / 2;
  static constexpr int kNPp = kNP | 1;  // odd stride (16-B units)
  static constexpr size_t kWarpBytes = (size_t)NB * kNPp * 16 + (size_t)NB * kC1 * 8;
  static constexpr int kFit = (int)((227 * 1024) / kWarpBytes);
  // warps per CTA: what shared memory holds, at most 12 (three per SM
  // sub-partition keep 168 registers per thread) -- 8 for cap 14, whose
  // 16-triple accumulators need more registers
  static constexpr int kMaxW = PRUNE ? (CAP >= 14 ? 8 : 12) : 16;
  static constexpr int kW = kFit < kMaxW ? kFit : kMaxW;
  // table index of pair (l, m): PRUNE m-major with m (CAP + 2 - m) before m
  static __host__ __device__ constexpr int pair(int l, int m) {
    return PRUNE ? m * (CAP + 2 - m) + (l - m) : l * (l + 1) / 2 + m;
  }
};

// PRUNE: the plan's labels all satisfy l + |m| <= CAP (true for every O3
// label a p = 1 target can use: the other factors must cancel m, and each
// costs at least its |m| of degree), so the table holds 49 of 91 pairs at
// cap 12 -- half the table work and a smaller table, hence more warps.
template <int CAP, int TPL, bool PRUNE>
__global__ void __launch_bounds__(Pool4Geom<CAP, PRUNE>::kW * 32, 1)
pool_positions4(const double* __restrict__ xyz, const int32_t* __restrict__ counts, int64_t S, int J, double r_in,
                double r_cut, const int4* __restrict__ tri, int ntri, const int32_t* __restrict__ col_of,
                int64_t out_stride, double2* __restrict__ out) {
  using G = Pool4Geom<CAP, PRUNE>;
  constexpr int C1 = G::kC1, NPp = G::kNPp, W = G::kW, NB = G::kNB;
  extern __shared__ __align__(16) unsigned char psm[];
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5);  // warp-uniform, told to the compiler
  double2* Y = reinterpret_cast<double2*>(psm + G::kWarpBytes * warp);  // [NB][NPp]
  double* WR = reinterpret_cast<double*>(Y + NB * NPp);                 // [NB][C1]
  const double inv_span = 1.0 / (r_cut - r_in);
  int tq[TPL];  // this lane's triples: pair << 8 | n (-1: none)
  // output columns of each triple and of its m -> -m partner (-1: not
  // wanted), looked up once: the site loop then stores without dependent
  // global loads
  int cpos[TPL], cneg[TPL];
#pragma unroll
  for (int t = 0; t < TPL; ++t) {
    const int i = lane + 32 * t;
    tq[t] = -1;
    cpos[t] = cneg[t] = -1;
    if (i < ntri) {
      const int4 q = __ldg(tri + i);
      tq[t] = G::pair(q.y, q.z) << 8 | q.x;
      cpos[t] = col_of ? col_of[q.w] : q.w;
      if (q.z > 0) cneg[t] = (col_of ? col_of[q.w - 2 * q.z] : q.w - 2 * q.z) | (q.z & 1) << 30;
    }
  }
  for (int64_t s = (int64_t)blockIdx.x * W + warp; s < S; s += (int64_t)gridDim.x * W) {
    const int nj = counts ? (int)uni((uint32_t)min(max(counts[s], 0), J)) : J;
    double2 acc[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) acc[t] = make_double2(0.0, 0.0);
    for (int j0 = 0; j0 < nj; j0 += NB) {
      const int nb = min(NB, nj - j0);
      if (lane < nb) {
        const double* p = xyz + (s * J + j0 + lane) * 3;
        const double x = p[0], y = p[1], z = p[2];
        const double rho2 = x * x + y * y;
        const double r = sqrt(rho2 + z * z);
        const double w = r < r_cut ? 0.5 * (1.0 + cospi(r / r_cut)) : 0.0;
        const double u = 2.0 * fmin(1.0, fmax(0.0, (r - r_in) * inv_span)) - 1.0;
        double* wr = WR + lane * C1;
        {
          double t0 = 1.0, t1 = u;
          wr[0] = w;
          if (CAP >= 1) wr[1] = w * u;
#pragma unroll
          for (int n = 2; n <= CAP; ++n) {
            const double t2 = 2.0 * u * t1 - t0;
            wr[n] = w * t2;
            t0 = t1;
            t1 = t2;
          }
        }
        const double rho = sqrt(rho2);
        const double ct = r > 0.0 ? z / r : 1.0, st = r > 0.0 ? rho / r : 0.0;
        const double cp = rho > 0.0 ? x / rho : 1.0, sp = rho > 0.0 ? y / rho : 0.0;
        double2* yj = Y + lane * NPp;
        double ec = 1.0, es = 0.0, pmm = 1.0;
        // l runs to LM(m): CAP, or CAP - m when the table is pruned
#pragma unroll
        for (int m = 0; m <= (PRUNE ? CAP / 2 : CAP); ++m) {
          constexpr int kLm0 = CAP;
          const int LM = PRUNE ? kLm0 - m : kLm0;
          if (m > 0) {
            const double nc = ec * cp - es * sp;
            es = ec * sp + es * cp;
            ec = nc;
            pmm *= -(2.0 * m - 1.0) * st;
          }
          double nv = c_ylm_norm[m * (m + 1) / 2 + m] * pmm;
          yj[G::pair(m, m)] = make_double2(nv * ec, nv * es);
          if (m + 1 <= LM) {
            double p0 = pmm, p1 = ct * (2.0 * m + 1.0) * pmm;
            nv = c_ylm_norm[(m + 1) * (m + 2) / 2 + m] * p1;
            yj[G::pair(m + 1, m)] = make_double2(nv * ec, nv * es);
#pragma unroll
            for (int l = m + 2; l <= LM; ++l) {
              const double p2 = (ct * (2.0 * l - 1.0) * p1 - (l + m - 1.0) * p0) * c_recip[l - m];
              nv = c_ylm_norm[l * (l + 1) / 2 + m] * p2;
              yj[G::pair(l, m)] = make_double2(nv * ec, nv * es);
              p0 = p1;
              p1 = p2;
            }
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < TPL; ++t) {
        if (tq[t] >= 0) {
          const int n = tq[t] & 255, pair = tq[t] >> 8;
          const double2* yp = Y + pair;
          const double* wp = WR + n;
          double ax = acc[t].x, ay = acc[t].y;
#pragma unroll 4
          for (int jj = 0; jj < nb; ++jj) {
            const double2 yv = yp[jj * NPp];
            const double a = wp[jj * C1];
            ax += a * yv.x;
            ay += a * yv.y;
          }
          acc[t] = make_double2(ax, ay);
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < TPL; ++t) {
      if (cpos[t] >= 0) out[s * out_stride + cpos[t]] = acc[t];
      const int cm = cneg[t] & 0x3FFFFFFF;
      if (cneg[t] >= 0 && cm != 0x3FFFFFFF) {  // A[n, l, -m] = (-1)^m conj(A[n, l, m])
        const double sg = (cneg[t] >> 30) & 1 ? -1.0 : 1.0;
        out[s * out_stride + cm] = make_double2(sg * acc[t].x, -sg * acc[t].y);
      }
    }
  }
}

// --------------------------------------------- K1 v5: accumulation on DMMA
// Per site the pooled basis is a small matrix product,
//     A[n][(l, m)] = sum_j WR[j][n] * Y[j][(l, m)],
// so v5 keeps v4's table phase (lane = neighbour, 16 neighbours per pass,
// pruned pairs l + m <= CAP) and runs the accumulation as
// mma.sync.m8n8k4.f64 tiles on the FP64 tensor cores: M = the radial index n
// (two 8-row tiles), N = the (re, im) columns of the pairs, K = the pass's 16
// neighbours.  Tables are stored j-fastest with a 20-entry j stride, which
// keeps both the table writes (lane = j) and the fragment loads free of bank
// conflicts.  Each warp keeps its site's [16 x 104] accumulator tile in
// registers (52 doubles per lane) across the passes; the lane that holds an
// (n, pair) element writes A[n, l, m] and A[n, l, -m] = (-1)^m conj(...).
// (One pass of 32 neighbours -- every lane in the table phase, 6 warps --
// ran cfg3 at 32.8 vs 30.9 ms per step with the k loop unrolled (spills),
// and at 28.75 vs 28.42 ms with it rolled.)
template <int CAP>
struct Pool5Geom {
  static constexpr int kNB = 16;                                     // neighbours per pass (K)
  static constexpr int kNJ = 20;                                     // j stride of the tables
  static constexpr int kC1 = CAP + 1;
  static constexpr int kMT = (kC1 + 7) / 8;                          // 8-row tiles of n
  static constexpr int kNP = (CAP / 2 + 1) * (CAP + 1 - CAP / 2);    // pairs with l + m <= CAP
  static constexpr int kNT = (2 * kNP + 7) / 8;                      // 8-column tiles of (re, im)
  // table rows kept in shared memory: the padding rows of the last tiles
  // (n past CAP, pairs past kNP) all read ONE zero row
  static constexpr int kRows = kNP < kNT * 4 ? kNP + 1 : kNT * 4;    // pair rows (+ the zero row)
  static constexpr int kWRows = kC1 < kMT * 8 ? kC1 + 1 : kMT * 8;   // radial rows (+ the zero row)
  static constexpr size_t kWarpBytes = (size_t)kRows * kNJ * 16 + (size_t)kWRows * kNJ * 8;
  // warps per CTA: as many as shared memory holds (18.2 KB per warp at cap
  // 12, 22.9 KB at cap 14); ptxas needs ~165 registers, so 12 x 168 / 9 x 224
  // fit without spills (cfg3 pool: 8 warps 8.35 ms per 1e6 sites, 10 8.08, 11 7.67)
  static constexpr int kW = CAP <= 12 ? 12 : 9;
  static constexpr size_t kOutBytes = (size_t)kMT * kNT * 32 * 8;    // per-lane output columns
  static constexpr size_t kSmem = (size_t)kW * kWarpBytes + kOutBytes;
  // pair index of (l, m), m-major (m = 0 first): l from m to CAP - m
  static __host__ __device__ constexpr int pair(int l, int m) { return m * (CAP + 2 - m) + (l - m); }
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// col_of: label -> output column (-1: unused); requires J passes of <= 16
// neighbours and a plan whose labels all satisfy l + |m| <= CAP
// tile_rows > 0: write straight into K2's tile-major seed table
// [S/128][tile_rows][128] (row = output column; row tile_rows - 1 = the
// constant ONE) instead of the site-major [S][out_stride] workspace, so the
// positions path needs no k_tile_seeds pass
template <int CAP>
__global__ void __launch_bounds__(Pool5Geom<CAP>::kW * 32, 1)
pool_positions5(const double* __restrict__ xyz, const int32_t* __restrict__ counts, int64_t S, int J, double r_in,
                double r_cut, const int32_t* __restrict__ col_of, int64_t out_stride, double2* __restrict__ out,
                int tile_rows) {
  using G = Pool5Geom<CAP>;
  constexpr int NJ = G::kNJ, NB = G::kNB, MT = G::kMT, NT = G::kNT, C1 = G::kC1, W = G::kW;
  extern __shared__ __align__(16) unsigned char psm[];
  const int lane = threadIdx.x & 31, warp = (int)uni(threadIdx.x >> 5);  // warp-uniform, told to the compiler
  double2* Y = reinterpret_cast<double2*>(psm + G::kWarpBytes * warp);  // [kRows][NJ]
  double* WR = reinterpret_cast<double*>(Y + G::kRows * NJ);            // [MT * 8][NJ]
  int2* ocol = reinterpret_cast<int2*>(psm + G::kWarpBytes * W);        // [MT][NT][32]
  // output columns of every accumulator element, per lane (same for all sites):
  // .x = column of (n, l, m), .y = column of (n, l, -m) | sign bit 30 (-1: none)
  for (int e = threadIdx.x; e < MT * NT * 32; e += blockDim.x) {
    const int ln = e & 31, nt = (e >> 5) % NT, mt = (e >> 5) / NT;
    const int n = mt * 8 + (ln >> 2), p = nt * 4 + (ln & 3);
    int2 oc = make_int2(-1, -1);
    if (n <= CAP && p < G::kNP) {
      int m = 0;
      while (m < CAP / 2 && p >= G::pair(m + 1, m + 1)) ++m;
      const int l = p - G::pair(m, m) + m;
      if (l + n <= CAP) {
        int base = 0;  // labels before n: sum over n' < n of (CAP - n' + 1)^2
        for (int q = 0; q < n; ++q) base += (CAP - q + 1) * (CAP - q + 1);
        const int lab = base + l * l + l + m;
        oc.x = col_of ? col_of[lab] : lab;
        if (m > 0) {
          const int cm = col_of ? col_of[lab - 2 * m] : lab - 2 * m;
          if (cm >= 0) oc.y = cm | (m & 1) << 30;
        }
      }
    }
    ocol[e] = oc;
  }
  __syncthreads();
  const double inv_span = 1.0 / (r_cut - r_in);
  for (int64_t s = (int64_t)blockIdx.x * W + warp; s < S; s += (int64_t)gridDim.x * W) {
    const int nj = counts ? (int)uni((uint32_t)min(max(counts[s], 0), J)) : J;
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int j0 = 0; j0 < nj; j0 += NB) {
      const int nb = min(NB, nj - j0);
      if (lane < NB) {
        const int jl = lane;
        if (jl < nb) {
          const double* p = xyz + (s * J + j0 + jl) * 3;
          const double x = p[0], y = p[1], z = p[2];
          const double rho2 = x * x + y * y;
          const double r = sqrt(rho2 + z * z);
          const double w = r < r_cut ? 0.5 * (1.0 + cospi(r / r_cut)) : 0.0;
          const double u = 2.0 * fmin(1.0, fmax(0.0, (r - r_in) * inv_span)) - 1.0;
          {
            double t0 = 1.0, t1 = u;
            WR[0 * NJ + jl] = w;
            if (CAP >= 1) WR[1 * NJ + jl] = w * u;
#pragma unroll
            for (int n = 2; n <= CAP; ++n) {
              const double t2 = 2.0 * u * t1 - t0;
              WR[n * NJ + jl] = w * t2;
              t0 = t1;
              t1 = t2;
            }
          }
          const double rho = sqrt(rho2);
          const double ct = r > 0.0 ? z / r : 1.0, st = r > 0.0 ? rho / r : 0.0;
          const double cp = rho > 0.0 ? x / rho : 1.0, sp = rho > 0.0 ? y / rho : 0.0;
          double ec = 1.0, es = 0.0, pmm = 1.0;
#pragma unroll
          for (int m = 0; m <= CAP / 2; ++m) {
            if (m > 0) {
              const double nc = ec * cp - es * sp;
              es = ec * sp + es * cp;
              ec = nc;
              pmm *= -(2.0 * m - 1.0) * st;
            }
            // the recurrence runs on the finished values Y = N P e^{i m phi}
            // (the phase is constant in l): five FP64 operations per (l, m)
            // pair instead of eight
            const double q0 = c_ylm_norm[m * (m + 1) / 2 + m] * pmm;
            double r0 = q0 * ec, i0 = q0 * es;
            Y[G::pair(m, m) * NJ + jl] = make_double2(r0, i0);
            if (m + 1 <= CAP - m) {
              const double a1 = c_ylm_a[(m + 1) * (m + 2) / 2 + m] * ct;
              double r1 = a1 * r0, i1 = a1 * i0;
              Y[G::pair(m + 1, m) * NJ + jl] = make_double2(r1, i1);
#pragma unroll
              for (int l = m + 2; l <= CAP - m; ++l) {
                const double al = c_ylm_a[l * (l + 1) / 2 + m] * ct, bl = c_ylm_b[l * (l + 1) / 2 + m];
                const double r2 = al * r1 - bl * r0, i2 = al * i1 - bl * i0;
                Y[G::pair(l, m) * NJ + jl] = make_double2(r2, i2);
                r0 = r1;
                i0 = i1;
                r1 = r2;
                i1 = i2;
              }
            }
          }
        } else {  // K padding of a short pass: zero weights and finite values
#pragma unroll
          for (int n = 0; n < G::kWRows; ++n) WR[n * NJ + jl] = 0.0;
          for (int q = 0; q < G::kRows; ++q) Y[q * NJ + jl] = make_double2(0.0, 0.0);
        }
      } else if (j0 == 0) {  // the zero rows (n past CAP, pairs past kNP): once per site
        for (int q = lane - NB; q < (G::kWRows - C1) * NB; q += 32 - NB)
          WR[(C1 + q / NB) * NJ + q % NB] = 0.0;
        for (int q = lane - NB; q < (G::kRows - G::kNP) * NB; q += 32 - NB)
          Y[(G::kNP + q / NB) * NJ + q % NB] = make_double2(0.0, 0.0);
      }
      __syncwarp();
      // the pass as 4 k-steps of 4 neighbours
#pragma unroll
      for (int ks = 0; ks < NB / 4; ++ks) {
        const int jj = ks * 4 + (lane & 3);
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          int row = mt * 8 + (lane >> 2);
          if (mt == MT - 1) row = min(row, G::kWRows - 1);  // padding rows -> the zero row
          a[mt] = WR[row * NJ + jj];
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int col = nt * 8 + (lane >> 2);
          int pr = col >> 1;
          if (nt == NT - 1) pr = min(pr, G::kRows - 1);  // padding pairs -> the zero row
          const double b = reinterpret_cast<const double*>(Y + pr * NJ + jj)[col & 1];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt][nt], a[mt], b);
        }
      }
      __syncwarp();
    }
    // site s, column c -> out[o0 + c * ostep]
    const int64_t o0 = tile_rows > 0 ? (s >> 7) * (int64_t)tile_rows * 128 + (s & 127) : s * out_stride;
    const int64_t ostep = tile_rows > 0 ? 128 : 1;
    if (tile_rows > 0 && lane == 0) out[o0 + (int64_t)(tile_rows - 1) * 128] = make_double2(1.0, 0.0);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int2 oc = ocol[(mt * NT + nt) * 32 + lane];
        if (oc.x >= 0) out[o0 + oc.x * ostep] = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        if (oc.y >= 0) {
          const double sg = (oc.y >> 30) & 1 ? -1.0 : 1.0;
          out[o0 + (oc.y & 0x3FFFFFFF) * ostep] = make_double2(sg * acc[mt][nt][0], -sg * acc[mt][nt][1]);
        }
      }
  }
}

}  // namespace dev
}  // namespace acedag
