// mf_common.cuh -- shared device helpers for the B200 assembly kernels.
//
// Classification and point-geometry arithmetic go through the *_rn
// intrinsics below so ptxas can never contract them into FMAs: the
// reference evaluates them unfused (numba build, SURVEY.md section 0 fact
// 4) and strict `<` tests on recursively bisected boxes must come out
// bit-identical (_kernels.py:80-102, 224-302).  Integrand arithmetic
// (mollifier value, weights, contractions) is free to use DFMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mollifem_b200.h"

#define MF_DEV __device__ __forceinline__

MF_DEV double xadd(double a, double b) { return __dadd_rn(a, b); }
MF_DEV double xsub(double a, double b) { return __dsub_rn(a, b); }
MF_DEV double xmul(double a, double b) { return __dmul_rn(a, b); }
MF_DEV double xdiv(double a, double b) { return __ddiv_rn(a, b); }
MF_DEV double xsqrt(double a) { return __dsqrt_rn(a); }
// Python min/max semantics (first argument wins ties)
MF_DEV double pmin(double a, double b) { return (b < a) ? b : a; }
MF_DEV double pmax(double a, double b) { return (b > a) ? b : a; }

// Everything one assembly launch needs, passed by value.
struct AsmParams {
  MfMesh mesh;
  MfRules rules;
  MfPattern pat;
  const uint8_t *outer_mask;
  const int32_t *inner;  // elements of the current colour
  int64_t n_inner;
  int32_t R;
  double scale;
  double *vals;
  unsigned long long *counters;
  int32_t flags;
  int32_t L_min, L_max;
  double delta, eps, cde;
  double dme, dpe;        // delta -/+ eps  (_kernels.py:410-411)
  double dm2, dp2;        // squared        (_kernels.py:412-413)
  double dme2_lo, dme2_hi;// sqrt-free decision band for aprx_max < dme
  double inv_eps, alpha;  // 1/eps and delta/eps (eps > 0 kernels)
  double alpha2;          // 2 delta/eps
  double half_inv_eps;    // 0.5/eps
  int32_t hi_dm2, hi_dp2; // high 32-bit words of dm2 / dp2 (non-negative
                          // doubles order like their bit patterns)
  int32_t hq_lo, hq_hi;   // high words of the shell edges (alpha -/+ 1)^2
                          // of q = d^2/eps^2, widened by one unit
  int32_t hd_lo, hd_hi;   // the same for d^2 itself: hi_dm2 - 1, hi_dp2 + 1
  int32_t nl_box, nl_tri;
  int32_t shortcuts;      // plateau/dead event shortcuts enabled
  double *scratch;        // per-thread scratch (generic kernel)
  int64_t scratch_stride; // doubles per thread
  int32_t *overflow;      // set when a specialised kernel cannot proceed
  // explicit pair lists (mf_general_core_lists, generic kernel only):
  // inner element inner[t] pairs with outer list_outer[k] for k in
  // [list_begin[t], list_end[t]); NULL = the cell-stencil product set
  const int64_t *list_begin, *list_end, *list_outer;
};

// aprx_min (_kernels.py:80-90): largest single-axis gap, 0 when overlapping
template <int DIM>
MF_DEV double aprx_min_d(const double *alo, const double *ahi,
                         const double *blo, const double *bhi) {
  double m = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    double d1 = xsub(alo[k], bhi[k]);
    double d2 = xsub(blo[k], ahi[k]);
    if (d1 > m) m = d1;
    if (d2 > m) m = d2;
  }
  return m;
}

// sum of per-axis max squared separations (argument of aprx_max's sqrt,
// _kernels.py:93-102), accumulated in the reference order without FMA
template <int DIM>
MF_DEV double aprx_max_sq(const double *alo, const double *ahi,
                          const double *blo, const double *bhi) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    double d1 = xsub(alo[k], bhi[k]);
    double d2 = xsub(blo[k], ahi[k]);
    double a = xmul(d1, d1), b = xmul(d2, d2);
    s = xadd(s, (a > b) ? a : b);
  }
  return s;
}

// sqrt(s) < dme, decided without the sqrt outside a 1e-12 relative band
// around dme^2 and with the correctly rounded sqrt inside it: same answer
// as the reference's `_aprx_max(...) < dme` for every s.
MF_DEV bool aprx_max_lt_dme(const AsmParams &P, double s) {
  if (s <= P.dme2_lo) return true;
  if (s >= P.dme2_hi) return false;
  return xsqrt(s) < P.dme;
}

// exact Euclidean box gap^2 >= dpe^2 test (dead-event proof; every point
// pair of the two boxes is then at distance >= delta+eps, so the
// reference skips all of them, _kernels.py:134-135).  Uses a relative
// safety margin so rounding can never prove a live event dead.
template <int DIM>
MF_DEV bool box_dead(const AsmParams &P, const double *alo, const double *ahi,
                     const double *blo, const double *bhi) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    // compare-and-select, not fmax: its NaN handling doubles the
    // instruction count on sm_100a and no NaN can occur here
    double g = pmax(alo[k] - bhi[k], blo[k] - ahi[k]);
    g = pmax(g, 0.0);
    s += g * g;
  }
  return s >= P.dp2 * (1.0 + 1e-9);
}

// mollifier value from the squared distance (_kernels.py:18-29) without
// the final /256 and the C constant (folded into weights by callers)
MF_DEV double xi_shell_256(const AsmParams &P, double d2) {
  double r = (P.delta - sqrt(d2)) / P.eps;
  double r2 = r * r;
  double p = fma(fma(fma(fma(35.0, r2, -180.0), r2, 378.0), r2, -420.0), r2,
                 315.0);
  return fma(p, r, 128.0);
}

// 1/x for normal x without the IEEE-division slow path (Newton twice)
MF_DEV double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// xi256 for N squared distances with ONE Newton correction folded into r:
// y = rsqrt(d2) (MUFU), d0 = d2 y, e0 = d2 - d0^2, and
//   r = (alpha - inv_eps d0) - (0.5 inv_eps y) e0
// which is alpha - inv_eps (d0 + 0.5 y e0), the Newton-corrected distance.
// Relative error of the distance ~ (rsqrt seed error)^2; 10 DP operations
// and 9 dependent levels instead of 12 and 13.
template <int N>
MF_DEV void xi256_fast_n(const AsmParams &P, const double *d2, double *out) {
  double y[N], d0[N], g[N], e[N], r[N];
#pragma unroll
  for (int i = 0; i < N; i++)
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[i]) : "d"(d2[i]));
#pragma unroll
  for (int i = 0; i < N; i++) {
    d0[i] = d2[i] * y[i];
    g[i] = P.half_inv_eps * y[i];
  }
#pragma unroll
  for (int i = 0; i < N; i++) {
    e[i] = fma(-d0[i], d0[i], d2[i]);
    r[i] = fma(-d0[i], P.inv_eps, P.alpha);
  }
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = fma(-g[i], e[i], r[i]);
  double r2[N], p[N];
#pragma unroll
  for (int i = 0; i < N; i++) r2[i] = r[i] * r[i];
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(35.0, r2[i], -180.0);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], 378.0);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], -420.0);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], 315.0);
#pragma unroll
  for (int i = 0; i < N; i++) out[i] = fma(p[i], r[i], 128.0);
}

// 256 mu(d) for N squared distances, eps > 0, with no classification:
// the high word of d2 is clamped to the shell [(delta-eps)^2,
// (delta+eps)^2] (widened by one unit) with integer min/max -- xi(+-1) =
// 256 / 0 with four vanishing derivatives, so the 2^-20 slack changes
// nothing above 1e-21 -- then one MUFU rsqrt seed z and the Newton step
// with its constants folded:  W = d2 z,  T = 3 - W z,  2 r = 2 alpha -
// (W T) / eps,  and xi as a polynomial in 2 r (coefficients 315/2, -420/8,
// 378/32, -180/128, 35/512, all exact).  10 DP operations, 2 integer, no
// selects, no vote.  (B200: FP64 and integer-ALU instructions hold the
// dispatch port for 2 cycles, so the selects of a classified form cost as
// much as the polynomial they avoid.)
template <int N>
MF_DEV void xi256_clamped_n(const AsmParams &P, const double *d2,
                            double *out) {
  double dc[N], z[N], W[N], T[N], r[N], r2[N], p[N];
#pragma unroll
  for (int i = 0; i < N; i++) {
    int hi = __double2hiint(d2[i]);
    hi = min(max(hi, P.hd_lo), P.hd_hi);
    dc[i] = __hiloint2double(hi, __double2loint(d2[i]));
  }
#pragma unroll
  for (int i = 0; i < N; i++)
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(z[i]) : "d"(dc[i]));
#pragma unroll
  for (int i = 0; i < N; i++) W[i] = dc[i] * z[i];
#pragma unroll
  for (int i = 0; i < N; i++) T[i] = fma(-W[i], z[i], 3.0);
#pragma unroll
  for (int i = 0; i < N; i++) W[i] = W[i] * T[i];
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = fma(-W[i], P.inv_eps, P.alpha2);
#pragma unroll
  for (int i = 0; i < N; i++) r2[i] = r[i] * r[i];
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(0.068359375, r2[i], -1.40625);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], 11.8125);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], -52.5);
#pragma unroll
  for (int i = 0; i < N; i++) p[i] = fma(p[i], r2[i], 157.5);
#pragma unroll
  for (int i = 0; i < N; i++) out[i] = fma(p[i], r[i], 128.0);
}

MF_DEV double mu256(const AsmParams &P, double d2) {
  if (d2 <= P.dm2) return 256.0;
  if (d2 >= P.dp2) return 0.0;
  return xi_shell_256(P, d2);
}

// flat pattern index of entry (r, c) (_eidx, _kernels.py:846-868)
MF_DEV int64_t pat_index(const MfPattern &p, int64_t r, int64_t c) {
  int NX = p.NX, NY = p.NY, K = p.K;
  int rx = (int)(r % NX);
  int64_t t = r / NX;
  int ry = (int)(t % NY), rz = (int)(t / NY);
  int cx = (int)(c % NX);
  int64_t u = c / NX;
  int cy = (int)(u % NY), cz = (int)(u / NY);
  int xlo = max(rx - K, 0), xhi = min(rx + K, NX - 1);
  int ylo = max(ry - K, 0), yhi = min(ry + K, NY - 1);
  int zlo = max(rz - K, 0);
  int Wx = xhi - xlo + 1, Wy = yhi - ylo + 1;
  return p.rowptr[r] + ((int64_t)(cz - zlo) * Wy + (cy - ylo)) * Wx +
         (cx - xlo);
}

MF_DEV void cell_coords(int c, int ncx, int ncy, int &cx, int &cy, int &cz) {
  cx = c % ncx;
  int t = c / ncx;
  cy = t % ncy;
  cz = t / ncy;
}

// max-axis gap between element boxes (outer l, inner e), exactly as
// _count_candidates (_kernels.py:1225-1233)
template <int DIM>
MF_DEV double elem_gap(const double *lo, const double *hi, int64_t l,
                       int64_t e) {
  double gap = 0.0;
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    double d1 = xsub(lo[l * DIM + k], hi[e * DIM + k]);
    double d2 = xsub(lo[e * DIM + k], hi[l * DIM + k]);
    if (d1 > gap) gap = d1;
    if (d2 > gap) gap = d2;
  }
  return gap;
}

// 1D Lagrange shapes on [-1,1] (_kernels.py:32-40)
MF_DEV void shape1d(int degree, double t, double *out) {
  if (degree == 1) {
    out[0] = 0.5 * (1.0 - t);
    out[1] = 0.5 * (1.0 + t);
  } else {
    out[0] = 0.5 * t * (t - 1.0);
    out[1] = 1.0 - t * t;
    out[2] = 0.5 * t * (t + 1.0);
  }
}

// shape values at reference coords (_kernels.py:43-77); returns nloc
MF_DEV int shape_at(int kind, int degree, int dim, double r0, double r1,
                    double r2, double *out) {
  if (kind == 1) {
    double la = 1.0 - r0 - r1;
    if (degree == 1) {
      out[0] = la;
      out[1] = r0;
      out[2] = r1;
      return 3;
    }
    out[0] = la * (2.0 * la - 1.0);
    out[1] = r0 * (2.0 * r0 - 1.0);
    out[2] = r1 * (2.0 * r1 - 1.0);
    out[3] = 4.0 * la * r0;
    out[4] = 4.0 * r0 * r1;
    out[5] = 4.0 * r1 * la;
    return 6;
  }
  double s0[3], s1[3], s2[3];
  int m = degree + 1, n = 0;
  shape1d(degree, r0, s0);
  shape1d(degree, r1, s1);
  if (dim == 2) {
    for (int j = 0; j < m; j++)
      for (int i = 0; i < m; i++) out[n++] = s0[i] * s1[j];
    return n;
  }
  shape1d(degree, r2, s2);
  for (int k = 0; k < m; k++)
    for (int j = 0; j < m; j++)
      for (int i = 0; i < m; i++) out[n++] = s0[i] * s1[j] * s2[k];
  return n;
}

// warp-aggregated counter add
MF_DEV void counter_add(unsigned long long *c, unsigned long long v) {
  if (v) atomicAdd(c, v);
}
