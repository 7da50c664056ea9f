// mf_2d.cu -- specialised adaptive assembly for pure 2D meshes of degree 1.
//
// Covers BASELINE config #1/#3 stand-ins: right
// triangle P1 with the Dunavant-7 rule (quadrature.py:141-142), and quad Q1
// with tensor Gauss/Lobatto rules of <= 4 (outer) / 3 (inner) points per
// axis; L_max <= 6.
//
// One thread per INNER element m of the current colour.  A 2D event is
// small (49 point pairs for triangles), so a whole pair fits one thread:
// the inner points y_q1, the per-pair accumulators
//   V[q1][j] = sum_events sum_q2 gamma(x_q2, y_q1) w_q2 phi_j(x_q2)
// and the element-level G[q1] = sum_pairs sum_j V[q1][j] live in registers.
// The partner loop walks the full, unclipped (2R+1)^2 stencil in the same
// order in every thread; same-colour elements handled by one warp have the
// same proto and nearby cells, so they visit partners at identical offsets
// and take identical Algorithm-1 paths (translation invariance), keeping
// the warp converged.  Algorithm 1 is the reference's depth-first walk
// (_pair_blocks, _kernels.py:184-313) with one geometry per level and the
// reference's midpoint arithmetic; L_max events are split into dead /
// plateau / full exactly as in mf_hex.cu.
#include "mf_common.cuh"

namespace {

constexpr int kMaxLevels = 6;
#ifndef MF_TRI_QUEUE
#define MF_TRI_QUEUE 1
#endif
#ifndef MF_2D_MINB
#define MF_2D_MINB 2
#endif

template <int KIND>
struct Cfg;
template <>
struct Cfg<1> {  // triangle P1
  static constexpr int NL = 3;
  static constexpr int NCHILD = 4;
};
template <>
struct Cfg<0> {  // quad Q1
  static constexpr int NL = 4;
  static constexpr int NCHILD = 4;
};

// position of the n-th (n >= 1) set bit of m, which must have at least n
// set bits: popc binary search (5 steps; the __fns intrinsic is a long
// generic loop and was 7% of k_tri_q's instructions)
MF_DEV int nth_set_bit(unsigned m, int n) {
  int pos = 0;
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const int c = __popc(m & ((1u << h) - 1u));
    if (n > c) {
      n -= c;
      pos += h;
      m >>= h;
    }
  }
  return pos;
}

// sub-cell bbox (_kernels.py:214-222)
template <int KIND>
MF_DEV void sub_bbox(const double *g, double *lo, double *hi) {
  if (KIND == 1) {
    lo[0] = pmin(g[0], pmin(g[2], g[4]));
    hi[0] = pmax(g[0], pmax(g[2], g[4]));
    lo[1] = pmin(g[1], pmin(g[3], g[5]));
    hi[1] = pmax(g[1], pmax(g[3], g[5]));
  } else {
    lo[0] = g[0];
    lo[1] = g[1];
    hi[0] = g[2];
    hi[1] = g[3];
  }
}

template <int KIND>
MF_DEV void make_child(const double *g, int b, double *c) {
  if (KIND == 1) {
    const double m010 = xmul(0.5, xadd(g[0], g[2]));
    const double m011 = xmul(0.5, xadd(g[1], g[3]));
    const double m120 = xmul(0.5, xadd(g[2], g[4]));
    const double m121 = xmul(0.5, xadd(g[3], g[5]));
    const double m200 = xmul(0.5, xadd(g[4], g[0]));
    const double m201 = xmul(0.5, xadd(g[5], g[1]));
    switch (b) {
      case 0:
        c[0] = g[0]; c[1] = g[1]; c[2] = m010; c[3] = m011; c[4] = m200;
        c[5] = m201;
        break;
      case 1:
        c[0] = m010; c[1] = m011; c[2] = g[2]; c[3] = g[3]; c[4] = m120;
        c[5] = m121;
        break;
      case 2:
        c[0] = m200; c[1] = m201; c[2] = m120; c[3] = m121; c[4] = g[4];
        c[5] = g[5];
        break;
      default:
        c[0] = m010; c[1] = m011; c[2] = m120; c[3] = m121; c[4] = m200;
        c[5] = m201;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const double lo = g[k], hi = g[2 + k];
      const double mid = xmul(0.5, xadd(lo, hi));
      if ((b >> k) & 1) {
        c[k] = mid;
        c[2 + k] = hi;
      } else {
        c[k] = lo;
        c[2 + k] = mid;
      }
    }
    c[4] = 0.0;
    c[5] = 0.0;
  }
}

// local DOF offsets on the DOF grid (degree 1, fe_space.py:68-80):
// tri lower (sw, se, ne), tri upper (sw, ne, nw), quad tensor-lex
MF_DEV void dof_offset(int kind, int proto, int j, int &ox, int &oy) {
  if (kind == 1) {
    if (proto == 0) {
      ox = j == 0 ? 0 : 1;
      oy = j == 2 ? 1 : 0;
    } else {
      ox = j == 1 ? 1 : 0;
      oy = j == 0 ? 0 : 1;
    }
  } else {
    ox = j & 1;
    oy = j >> 1;
  }
}

struct OuterTri {
  double v0[2], inv[4];
};
struct OuterBox {
  double lo[2], inv[2];
};

// ---- triangle events (Dunavant outer rule in shared memory) ----
// VOTE: evaluate the shell polynomials only when some lane of the warp
// needs one (thread-per-pair callers, whose lanes hold unrelated pairs);
// the warp-cooperative phase B of k_tri_q passes false: there every lane
// integrates a full event and the vote nearly always fires (R2-small
// 186 -> 178 ms without it; k_2d on R3-16h is faster with it, 669 vs 725)
template <int NQO, int NQ1, bool SHARP, bool VOTE = true>
MF_DEV void tri_full(const AsmParams &P, const double *g, const OuterTri &O,
                     const double (*y)[2], const double *s_pts,
                     const double *s_w, double (*V)[3]) {
  const double e10 = xsub(g[2], g[0]), e11 = xsub(g[3], g[1]);
  const double e20 = xsub(g[4], g[0]), e21 = xsub(g[5], g[1]);
  const double det = e10 * e21 - e11 * e20;
  const double f = det * P.cde * (1.0 / 256.0);
#pragma unroll 1
  for (int q2 = 0; q2 < NQO; q2++) {
    const double px = s_pts[2 * q2], py = s_pts[2 * q2 + 1];
    // eps = 0: the reference's unfused order (ties); else two FMAs
    const double x0 = SHARP ? xadd(xadd(g[0], xmul(px, e10)), xmul(py, e20))
                            : fma(py, e20, fma(px, e10, g[0]));
    const double x1 = SHARP ? xadd(xadd(g[1], xmul(px, e11)), xmul(py, e21))
                            : fma(py, e21, fma(px, e11, g[1]));
    const double w2 = s_w[q2] * f;
    const double dx0 = x0 - O.v0[0], dx1 = x1 - O.v0[1];
    const double rx = O.inv[0] * dx0 + O.inv[1] * dx1;
    const double ry = O.inv[2] * dx0 + O.inv[3] * dx1;
    const double p1 = rx * w2, p2 = ry * w2, p0 = w2 - p1 - p2;
    double mu[NQ1];
    if (SHARP) {
#pragma unroll
      for (int q1 = 0; q1 < NQ1; q1++) {
        const double dx = xsub(x0, y[q1][0]), dy = xsub(x1, y[q1][1]);
        const double d2 = xadd(xmul(dx, dx), xmul(dy, dy));
        mu[q1] = d2 < P.dp2 ? 256.0 : 0.0;
      }
    } else {
      // eps > 0: mu is continuous, so the distances may use fused
      // arithmetic and the clamped mollifier needs no classification
      double d2[NQ1];
#pragma unroll
      for (int q1 = 0; q1 < NQ1; q1++) {
        const double dx = x0 - y[q1][0], dy = x1 - y[q1][1];
        d2[q1] = fma(dy, dy, dx * dx);
      }
      xi256_clamped_n<NQ1>(P, d2, mu);
    }
#pragma unroll
    for (int q1 = 0; q1 < NQ1; q1++) {
      V[q1][0] = fma(mu[q1], p0, V[q1][0]);
      V[q1][1] = fma(mu[q1], p1, V[q1][1]);
      V[q1][2] = fma(mu[q1], p2, V[q1][2]);
    }
  }
}

template <int NQO>
MF_DEV void tri_plateau(const AsmParams &P, const double *g,
                        const OuterTri &O, const double *s_pts,
                        const double *s_w, double *SP) {
  const double e10 = g[2] - g[0], e11 = g[3] - g[1];
  const double e20 = g[4] - g[0], e21 = g[5] - g[1];
  const double det = e10 * e21 - e11 * e20;
  const double f = det * P.cde;
#pragma unroll 1
  for (int q2 = 0; q2 < NQO; q2++) {
    const double px = s_pts[2 * q2], py = s_pts[2 * q2 + 1];
    const double x0 = g[0] + px * e10 + py * e20;
    const double x1 = g[1] + px * e11 + py * e21;
    const double w2 = s_w[q2] * f;
    const double dx0 = x0 - O.v0[0], dx1 = x1 - O.v0[1];
    const double rx = O.inv[0] * dx0 + O.inv[1] * dx1;
    const double ry = O.inv[2] * dx0 + O.inv[3] * dx1;
    SP[0] += w2 * (1.0 - rx - ry);
    SP[1] += w2 * rx;
    SP[2] += w2 * ry;
  }
}

// ---- quad events (tensor outer rule, sum-factorised) ----
template <int NO>
MF_DEV void box_axes(const AsmParams &P, const double *g, const OuterBox &O,
                     const double *s_t, const double *s_w, double X[2][NO],
                     double sh[2][2][NO]) {
  const double jac = (0.5 * (g[2] - g[0])) * (0.5 * (g[3] - g[1]));
  const double f0 = P.cde * jac * (1.0 / 256.0);
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const double wk = xsub(g[2 + k], g[k]);
#pragma unroll
    for (int a = 0; a < NO; a++) {
      const double x = xadd(g[k], xmul(s_t[a], wk));
      X[k][a] = x;
      const double s1 = (x - O.lo[k]) * O.inv[k];
      const double wa = s_w[a] * (k == 0 ? f0 : 1.0);
      sh[k][0][a] = (1.0 - s1) * wa;
      sh[k][1][a] = s1 * wa;
    }
  }
}

template <int NO, int NQ1, bool SHARP>
MF_DEV void quad_full(const AsmParams &P, const double *g, const OuterBox &O,
                      const double (*y)[2], const double *s_t,
                      const double *s_w, double (*V)[4]) {
  double X[2][NO], sh[2][2][NO];
  box_axes<NO>(P, g, O, s_t, s_w, X, sh);
#pragma unroll 1
  for (int q1 = 0; q1 < NQ1; q1++) {
    double sqx[NO], sqy[NO];
#pragma unroll
    for (int a = 0; a < NO; a++) {
      const double dx = xsub(X[0][a], y[q1][0]);
      const double dy = xsub(X[1][a], y[q1][1]);
      sqx[a] = xmul(dx, dx);
      sqy[a] = xmul(dy, dy);
    }
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
    for (int b = 0; b < NO; b++) {
      double mu[NO];
      if (SHARP) {
#pragma unroll
        for (int a = 0; a < NO; a++)
          mu[a] = xadd(sqx[a], sqy[b]) < P.dp2 ? 256.0 : 0.0;
      } else {
        double d2[NO];
#pragma unroll
        for (int a = 0; a < NO; a++) d2[a] = sqx[a] + sqy[b];
        xi256_clamped_n<NO>(P, d2, mu);
      }
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int a = 0; a < NO; a++) {
        t0 = fma(mu[a], sh[0][0][a], t0);
        t1 = fma(mu[a], sh[0][1][a], t1);
      }
      v0 = fma(t0, sh[1][0][b], v0);
      v1 = fma(t1, sh[1][0][b], v1);
      v2 = fma(t0, sh[1][1][b], v2);
      v3 = fma(t1, sh[1][1][b], v3);
    }
    // dynamic q1 index: V lives in local memory for this path
    V[q1][0] += v0;
    V[q1][1] += v1;
    V[q1][2] += v2;
    V[q1][3] += v3;
  }
}

template <int NO>
MF_DEV void quad_plateau(const AsmParams &P, const double *g,
                         const OuterBox &O, const double *s_t,
                         const double *s_w, double *SP) {
  double X[2][NO], sh[2][2][NO];
  box_axes<NO>(P, g, O, s_t, s_w, X, sh);
  double S[2][2];
#pragma unroll
  for (int k = 0; k < 2; k++)
#pragma unroll
    for (int j = 0; j < 2; j++) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < NO; a++) s += sh[k][j][a];
      S[k][j] = s;
    }
#pragma unroll
  for (int jy = 0; jy < 2; jy++)
#pragma unroll
    for (int jx = 0; jx < 2; jx++) SP[jx + 2 * jy] += 256.0 * S[0][jx] * S[1][jy];
}

enum : int { ACT_NONE = 0, ACT_SPLIT = 1, ACT_UPPER = 2, ACT_PLAT = 3,
             ACT_DEAD = 4, ACT_FULL = 5 };

// KIND 1: tri P1 with Dunavant (NO = NI = 7 points, unused template args)
// KIND 0: quad Q1 with NO / NI points per axis
template <int KIND, int NO, int NI>
__global__ void __launch_bounds__(128, MF_2D_MINB) k_2d(AsmParams P) {
  constexpr int NL = Cfg<KIND>::NL;
  constexpr int NQ1 = KIND == 1 ? 7 : NI * NI;
  constexpr int NQO = KIND == 1 ? 7 : NO;  // per-axis (quad) / total (tri)
  __shared__ double s_phiw[NQ1][NL], s_phi[NQ1][NL];
  __shared__ double s_opts[2 * NQO], s_ow[NQO];
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * NL; i += blockDim.x) {
    const int q = i / NL, j = i % NL;
    const double ph = KIND == 1 ? Rr.phi_tri_in[q * NL + j]
                                : Rr.phi_box_in[q * NL + j];
    s_phi[q][j] = ph;
    s_phiw[q][j] = (KIND == 1 ? Rr.tri_in_w[q] : Rr.box_in_w[q]) * ph;
  }
  for (int i = threadIdx.x; i < NQO; i += blockDim.x) {
    if (KIND == 1) {
      s_opts[2 * i] = Rr.tri_out_pts[2 * i];
      s_opts[2 * i + 1] = Rr.tri_out_pts[2 * i + 1];
      s_ow[i] = Rr.tri_out_w[i];
    } else {
      s_opts[i] = xmul(xadd(Rr.box_out_x1d[i], 1.0), 0.5);
      s_ow[i] = Rr.box_out_w1d[i];
    }
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.n_inner) return;
  const int64_t m = P.inner[t];

  // inner element: exact points (_inner_data) and measure factor
  double y[NQ1][2];
  double ilo[2], ihi[2], scale_in;
  ilo[0] = M.elem_lo[m * 2];
  ilo[1] = M.elem_lo[m * 2 + 1];
  ihi[0] = M.elem_hi[m * 2];
  ihi[1] = M.elem_hi[m * 2 + 1];
  if (KIND == 1) {
    const double *c = M.elem_coords + m * M.nv_max * 2;
    const double e10 = xsub(c[2], c[0]), e11 = xsub(c[3], c[1]);
    const double e20 = xsub(c[4], c[0]), e21 = xsub(c[5], c[1]);
    scale_in = e10 * e21 - e11 * e20;
#pragma unroll
    for (int q = 0; q < NQ1; q++) {
      const double p0 = Rr.tri_in_pts[2 * q], p1 = Rr.tri_in_pts[2 * q + 1];
      y[q][0] = xadd(xadd(c[0], xmul(p0, e10)), xmul(p1, e20));
      y[q][1] = xadd(xadd(c[1], xmul(p0, e11)), xmul(p1, e21));
    }
  } else {
    scale_in = (0.5 * (ihi[0] - ilo[0])) * (0.5 * (ihi[1] - ilo[1]));
#pragma unroll
    for (int q = 0; q < NQ1; q++)
#pragma unroll
      for (int k = 0; k < 2; k++)
        y[q][k] = xadd(ilo[k], xmul(xmul(xadd(Rr.box_in_pts[2 * q + k], 1.0),
                                         0.5),
                                    xsub(ihi[k], ilo[k])));
  }
  double G[NQ1];
#pragma unroll
  for (int q = 0; q < NQ1; q++) G[q] = 0.0;
  unsigned long long c_ev = 0, c_pairs = 0, c_up = 0, c_pl = 0, c_dead = 0,
                     c_full = 0;
  int cx, cy, cz;
  cell_coords(M.elem_cell[m], M.ncx, M.ncy, cx, cy, cz);
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
  const int Rs = P.R;
  // implicit-pattern geometry of this element's rows (assembly.py:197-223):
  // entry (r, c) = rowbase + (gy_c - ylo) * Wx + (gx_c - xlo)
  const int nproto = KIND == 1 ? 2 : 1;
  const int tin = (int)(m % nproto);
  int64_t rowbase[NL];
  int rxlo[NL], rylo[NL], rwx[NL];
#pragma unroll
  for (int i = 0; i < NL; i++) {
    int ox, oy;
    dof_offset(KIND, tin, i, ox, oy);
    const int gx = cx + ox, gy = cy + oy;
    rxlo[i] = max(gx - P.pat.K, 0);
    rwx[i] = min(gx + P.pat.K, P.pat.NX - 1) - rxlo[i] + 1;
    rylo[i] = max(gy - P.pat.K, 0);
    rowbase[i] = P.pat.rowptr[mdofs[i]];
  }

  for (int dy = -Rs; dy <= Rs; dy++) {
    const int y2 = cy + dy;
    if (y2 < 0 || y2 >= M.ncy) continue;
    for (int dx = -Rs; dx <= Rs; dx++) {
      const int x2 = cx + dx;
      if (x2 < 0 || x2 >= M.ncx) continue;
      const int64_t c2 = (int64_t)y2 * M.ncx + x2;
      for (int64_t l = M.cell_ptr[c2]; l < M.cell_ptr[c2 + 1]; l++) {
        if (!P.outer_mask[l]) continue;
        if (!(elem_gap<2>(M.elem_lo, M.elem_hi, l, m) < P.dpe)) continue;
        c_pairs++;
        // value slots of this pair's A21 block, prefetched into L2 now so
        // the read-modify-write at the end of the pair does not stall
        const int tout = (int)(l % nproto);
        int64_t slot[NL][NL];
#pragma unroll
        for (int j = 0; j < NL; j++) {
          int ox, oy;
          dof_offset(KIND, tout, j, ox, oy);
          const int gx = x2 + ox, gy = y2 + oy;
#pragma unroll
          for (int i = 0; i < NL; i++) {
            slot[i][j] = rowbase[i] + (int64_t)(gy - rylo[i]) * rwx[i] +
                         (gx - rxlo[i]);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot[i][j]));
          }
        }
        OuterTri OT;
        OuterBox OB;
        double root[6];
        if (KIND == 1) {
          const double *c = M.elem_coords + l * M.nv_max * 2;
#pragma unroll
          for (int u = 0; u < 6; u++) root[u] = c[u];
          const double e10 = c[2] - c[0], e11 = c[3] - c[1];
          const double e20 = c[4] - c[0], e21 = c[5] - c[1];
          const double det = e10 * e21 - e11 * e20;
          OT.v0[0] = c[0];
          OT.v0[1] = c[1];
          const double idet = rcp_fast(det);
          OT.inv[0] = e21 * idet;
          OT.inv[1] = -e20 * idet;
          OT.inv[2] = -e11 * idet;
          OT.inv[3] = e10 * idet;
        } else {
#pragma unroll
          for (int k = 0; k < 2; k++) {
            root[k] = M.elem_lo[l * 2 + k];
            root[2 + k] = M.elem_hi[l * 2 + k];
            OB.lo[k] = root[k];
            OB.inv[k] = rcp_fast(root[2 + k] - root[k]);
          }
          root[4] = root[5] = 0.0;
        }
        double V[NQ1][NL];
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
          for (int j = 0; j < NL; j++) V[q][j] = 0.0;
        double SP[NL];
#pragma unroll
        for (int j = 0; j < NL; j++) SP[j] = 0.0;
        unsigned long long ev = 0;
        bool live = false;  // some plateau/full event: nonzero block
        double geo[kMaxLevels + 1][6];
        int child[kMaxLevels + 1];
#pragma unroll
        for (int u = 0; u < 6; u++) geo[1][u] = root[u];
        int L = 1;
        for (;;) {
          double slo[2], shi[2];
          sub_bbox<KIND>(geo[L], slo, shi);
          int act = ACT_NONE;
          if (L < P.L_min) {
            act = ACT_SPLIT;
          } else if (L == P.L_max) {
            if (aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe) {
              if (!P.shortcuts)
                act = ACT_FULL;
              else if (box_dead<2>(P, slo, shi, ilo, ihi))
                act = ACT_DEAD;
              else if (aprx_max_lt_dme(P, aprx_max_sq<2>(slo, shi, ilo, ihi)))
                act = ACT_PLAT;
              else
                act = ACT_FULL;
            }
          } else if (aprx_max_lt_dme(P, aprx_max_sq<2>(slo, shi, ilo, ihi))) {
            act = ACT_UPPER;
          } else if (aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe) {
            act = ACT_SPLIT;
          }
          if (act >= ACT_UPPER) {
            ev++;
            if (act == ACT_UPPER) c_up++;
            if (act == ACT_DEAD) c_dead++;
            if (act == ACT_PLAT) c_pl++;
            if (act == ACT_FULL) c_full++;
            const bool plateau =
                act == ACT_PLAT || (act == ACT_UPPER && P.shortcuts);
            const bool full = act == ACT_FULL || (act == ACT_UPPER &&
                                                  !P.shortcuts);
            live |= plateau || full;
            if constexpr (KIND == 1) {
              if (plateau)
                tri_plateau<7>(P, geo[L], OT, s_opts, s_ow, SP);
              else if (full && P.eps > 0.0)
                tri_full<7, NQ1, false>(P, geo[L], OT, y, s_opts, s_ow,
                                     reinterpret_cast<double(*)[3]>(V));
              else if (full)
                tri_full<7, NQ1, true>(P, geo[L], OT, y, s_opts, s_ow,
                                    reinterpret_cast<double(*)[3]>(V));
            } else {
              if (plateau)
                quad_plateau<NO>(P, geo[L], OB, s_opts, s_ow, SP);
              else if (full && P.eps > 0.0)
                quad_full<NO, NQ1, false>(P, geo[L], OB, y, s_opts, s_ow,
                                          reinterpret_cast<double(*)[4]>(V));
              else if (full)
                quad_full<NO, NQ1, true>(P, geo[L], OB, y, s_opts, s_ow,
                                         reinterpret_cast<double(*)[4]>(V));
            }
          }
          if (act == ACT_SPLIT) {
            ++L;
            child[L] = 0;
            make_child<KIND>(geo[L - 1], 0, geo[L]);
            continue;
          }
          bool done = false;
          for (;;) {
            if (L == 1) {
              done = true;
              break;
            }
            if (++child[L] < Cfg<KIND>::NCHILD) {
              make_child<KIND>(geo[L - 1], child[L], geo[L]);
              break;
            }
            --L;
          }
          if (done) break;
        }
        c_ev += ev;
        // dead-only pairs add an exactly zero block: skipped
        if (live) {
          // plateau part is common to every q1
          double spsum = 0.0;
#pragma unroll
          for (int j = 0; j < NL; j++) spsum += SP[j];
          const double sc = -P.scale * scale_in;
          // old values loaded together before any store (overlapped
          // latencies; the compiler cannot prove the slots distinct)
          double old[NL][NL];
#pragma unroll
          for (int i = 0; i < NL; i++)
#pragma unroll
            for (int j = 0; j < NL; j++) old[i][j] = P.vals[slot[i][j]];
#pragma unroll
          for (int i = 0; i < NL; i++) {
            double mi = 0.0;
#pragma unroll
            for (int q = 0; q < NQ1; q++) mi += s_phiw[q][i];
#pragma unroll
            for (int j = 0; j < NL; j++) {
              double b = mi * SP[j];
#pragma unroll
              for (int q = 0; q < NQ1; q++) b = fma(s_phiw[q][i], V[q][j], b);
              P.vals[slot[i][j]] = old[i][j] + sc * b;
            }
          }
#pragma unroll
          for (int q = 0; q < NQ1; q++) {
            double s = spsum;
#pragma unroll
            for (int j = 0; j < NL; j++) s += V[q][j];
            G[q] += s;
          }
        }
      }
    }
  }
  // A22 of the element
  const double sc = P.scale * scale_in;
#pragma unroll
  for (int i = 0; i < NL; i++) {
    const int64_t r = mdofs[i];
#pragma unroll
    for (int j = 0; j < NL; j++) {
      double b = 0.0;
#pragma unroll
      for (int q = 0; q < NQ1; q++) b = fma(G[q] * s_phiw[q][i], s_phi[q][j], b);
      P.vals[pat_index(P.pat, r, mdofs[j])] += sc * b;
    }
  }
  unsigned long long *C = P.counters;
  counter_add(C + MF_CNT_EVENTS, c_ev);
  counter_add(C + MF_CNT_PAIRS, c_pairs);
  counter_add(C + MF_CNT_EV_UPPER, c_up);
  counter_add(C + MF_CNT_EV_PLATEAU, c_pl);
  counter_add(C + MF_CNT_EV_DEAD, c_dead);
  counter_add(C + MF_CNT_EV_FULL, c_full);
}

// ---- unstructured P1 triangles (mesh layout 1, BASELINE config #2) ----
//
// Delaunay triangles of any shape (mesh.py build_delaunay_mesh), binned by
// the lattice cell of their box lower corner; elem_dofs are lattice ids on
// the implicit pattern grid.  One thread = one INNER element m of the
// current colour (a greedy vertex-disjoint colouring) x ONE stencil bin
// row dy (blockIdx.y); a launch covers the rows of one class
// (dy + R) mod row_period.  Outer elements binned row_period rows apart
// share no vertex (emax <= (row_period - 1) h, checked by the mesh
// builder), and same-colour inner elements share no vertex, so the A21
// read-modify-writes of one launch never collide: no atomics, a fixed
// launch order, deterministic.  The outer elements of a bin row are one
// contiguous id range (bin-lex order).  Each thread leaves its G partial in
// gscr[row][element]; k_tri_u_a22 sums the rows in order and folds A22.
// Algorithm 1 and the events are those of k_2d<1> (the reference's
// _event_tri is valid for arbitrary affine triangles, _kernels.py:146-181).
template <int NQO, int NQ1>
__global__ void __launch_bounds__(128, MF_2D_MINB)
    k_tri_u(AsmParams P, int cls, double *gscr) {
  constexpr int NL = 3;
  __shared__ double s_phiw[NQ1][NL];
  __shared__ double s_opts[2 * NQO], s_ow[NQO];
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * NL; i += blockDim.x) {
    const int q = i / NL, j = i % NL;
    s_phiw[q][j] = Rr.tri_in_w[q] * Rr.phi_tri_in[q * NL + j];
  }
  for (int i = threadIdx.x; i < NQO; i += blockDim.x) {
    s_opts[2 * i] = Rr.tri_out_pts[2 * i];
    s_opts[2 * i + 1] = Rr.tri_out_pts[2 * i + 1];
    s_ow[i] = Rr.tri_out_w[i];
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.n_inner) return;
  const int Rs = P.R;
  const int pidx = cls + M.row_period * (int)blockIdx.y;  // dy + R
  const int dy = pidx - Rs;
  const int64_t m = P.inner[t];
  double G[NQ1];
#pragma unroll
  for (int q = 0; q < NQ1; q++) G[q] = 0.0;
  unsigned c_ev = 0, c_pairs = 0, c_up = 0, c_pl = 0, c_dead = 0, c_full = 0;
  const int cell = M.elem_cell[m];
  const int cx = cell % M.ncx, cy = cell / M.ncx;
  const int y2 = cy + dy;
  if (y2 >= 0 && y2 < M.ncy) {
    // inner element: exact points (_inner_data) and measure factor
    double y[NQ1][2];
    double ilo[2], ihi[2];
    ilo[0] = M.elem_lo[m * 2];
    ilo[1] = M.elem_lo[m * 2 + 1];
    ihi[0] = M.elem_hi[m * 2];
    ihi[1] = M.elem_hi[m * 2 + 1];
    double scale_in;
    {
      const double *c = M.elem_coords + m * M.nv_max * 2;
      const double e10 = xsub(c[2], c[0]), e11 = xsub(c[3], c[1]);
      const double e20 = xsub(c[4], c[0]), e21 = xsub(c[5], c[1]);
      scale_in = e10 * e21 - e11 * e20;
#pragma unroll
      for (int q = 0; q < NQ1; q++) {
        const double p0 = Rr.tri_in_pts[2 * q], p1 = Rr.tri_in_pts[2 * q + 1];
        y[q][0] = xadd(xadd(c[0], xmul(p0, e10)), xmul(p1, e20));
        y[q][1] = xadd(xadd(c[1], xmul(p0, e11)), xmul(p1, e21));
      }
    }
    // rows of the element's 3 vertices on the implicit pattern
    // (assembly.py:197-223): entry (r, c) = rowptr[r] + (gy_c - ylo) Wx +
    // (gx_c - xlo)
    const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
    const int NX = P.pat.NX, K = P.pat.K;
    int64_t rowbase[NL];
    int rxlo[NL], rylo[NL], rwx[NL];
#pragma unroll
    for (int i = 0; i < NL; i++) {
      const int d = (int)mdofs[i];
      const int gx = d % NX, gy = d / NX;
      rxlo[i] = max(gx - K, 0);
      rwx[i] = min(gx + K, NX - 1) - rxlo[i] + 1;
      rylo[i] = max(gy - K, 0);
      rowbase[i] = P.pat.rowptr[d];
    }
    const int64_t l0 = M.cell_ptr[(int64_t)y2 * M.ncx + max(cx - Rs, 0)];
    const int64_t l1 =
        M.cell_ptr[(int64_t)y2 * M.ncx + min(cx + Rs, M.ncx - 1) + 1];
    for (int64_t l = l0; l < l1; l++) {
      if (!P.outer_mask[l]) continue;
      if (!(elem_gap<2>(M.elem_lo, M.elem_hi, l, m) < P.dpe)) continue;
      c_pairs++;
      const int64_t *ldofs = M.elem_dofs + l * M.nloc_max;
      int64_t slot[NL][NL];
#pragma unroll
      for (int j = 0; j < NL; j++) {
        const int d = (int)ldofs[j];
        const int gx = d % NX, gy = d / NX;
#pragma unroll
        for (int i = 0; i < NL; i++) {
          slot[i][j] = rowbase[i] + (int64_t)(gy - rylo[i]) * rwx[i] +
                       (gx - rxlo[i]);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot[i][j]));
        }
      }
      OuterTri OT;
      double geo[kMaxLevels + 1][6];
      {
        const double *c = M.elem_coords + l * M.nv_max * 2;
#pragma unroll
        for (int u = 0; u < 6; u++) geo[1][u] = c[u];
        const double e10 = c[2] - c[0], e11 = c[3] - c[1];
        const double e20 = c[4] - c[0], e21 = c[5] - c[1];
        const double idet = rcp_fast(e10 * e21 - e11 * e20);
        OT.v0[0] = c[0];
        OT.v0[1] = c[1];
        OT.inv[0] = e21 * idet;
        OT.inv[1] = -e20 * idet;
        OT.inv[2] = -e11 * idet;
        OT.inv[3] = e10 * idet;
      }
      double V[NQ1][NL];
#pragma unroll
      for (int q = 0; q < NQ1; q++)
#pragma unroll
        for (int j = 0; j < NL; j++) V[q][j] = 0.0;
      double SP[NL] = {0.0, 0.0, 0.0};
      unsigned ev = 0;
      bool live = false;  // some plateau/full event: nonzero block
      int child[kMaxLevels + 1];
      int L = 1;
      for (;;) {
        double slo[2], shi[2];
        sub_bbox<1>(geo[L], slo, shi);
        int act = ACT_NONE;
        if (L < P.L_min) {
          act = ACT_SPLIT;
        } else if (L == P.L_max) {
          if (aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe) {
            if (!P.shortcuts)
              act = ACT_FULL;
            else if (box_dead<2>(P, slo, shi, ilo, ihi))
              act = ACT_DEAD;
            else if (aprx_max_lt_dme(P, aprx_max_sq<2>(slo, shi, ilo, ihi)))
              act = ACT_PLAT;
            else
              act = ACT_FULL;
          }
        } else if (aprx_max_lt_dme(P, aprx_max_sq<2>(slo, shi, ilo, ihi))) {
          act = ACT_UPPER;
        } else if (aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe) {
          act = ACT_SPLIT;
        }
        if (act >= ACT_UPPER) {
          ev++;
          if (act == ACT_UPPER) c_up++;
          if (act == ACT_DEAD) c_dead++;
          if (act == ACT_PLAT) c_pl++;
          if (act == ACT_FULL) c_full++;
          const bool plateau =
              act == ACT_PLAT || (act == ACT_UPPER && P.shortcuts);
          const bool full =
              act == ACT_FULL || (act == ACT_UPPER && !P.shortcuts);
          live |= plateau || full;
          if (plateau)
            tri_plateau<NQO>(P, geo[L], OT, s_opts, s_ow, SP);
          else if (full && P.eps > 0.0)
            tri_full<NQO, NQ1, false>(P, geo[L], OT, y, s_opts, s_ow, V);
          else if (full)
            tri_full<NQO, NQ1, true>(P, geo[L], OT, y, s_opts, s_ow, V);
        }
        if (act == ACT_SPLIT) {
          ++L;
          child[L] = 0;
          make_child<1>(geo[L - 1], 0, geo[L]);
          continue;
        }
        bool done = false;
        for (;;) {
          if (L == 1) {
            done = true;
            break;
          }
          if (++child[L] < 4) {
            make_child<1>(geo[L - 1], child[L], geo[L]);
            break;
          }
          --L;
        }
        if (done) break;
      }
      c_ev += ev;
      // dead-only pairs add an exactly zero block: skipped
      if (live) {
        const double spsum = (SP[0] + SP[1]) + SP[2];
        const double sc = -P.scale * scale_in;
        double old[NL][NL];
#pragma unroll
        for (int i = 0; i < NL; i++)
#pragma unroll
          for (int j = 0; j < NL; j++) old[i][j] = P.vals[slot[i][j]];
#pragma unroll
        for (int i = 0; i < NL; i++) {
          double mi = 0.0;
#pragma unroll
          for (int q = 0; q < NQ1; q++) mi += s_phiw[q][i];
#pragma unroll
          for (int j = 0; j < NL; j++) {
            double b = mi * SP[j];
#pragma unroll
            for (int q = 0; q < NQ1; q++) b = fma(s_phiw[q][i], V[q][j], b);
            P.vals[slot[i][j]] = old[i][j] + sc * b;
          }
        }
#pragma unroll
        for (int q = 0; q < NQ1; q++) {
          double sg = spsum;
#pragma unroll
          for (int j = 0; j < NL; j++) sg += V[q][j];
          G[q] += sg;
        }
      }
    }
  }
  double *gp = gscr + ((int64_t)pidx * P.n_inner + t) * NQ1;
#pragma unroll
  for (int q = 0; q < NQ1; q++) gp[q] = G[q];
  const unsigned mask = __activemask();
  const unsigned v[6] = {c_ev, c_pairs, c_up, c_pl, c_dead, c_full};
  const int cslot[6] = {MF_CNT_EVENTS, MF_CNT_PAIRS, MF_CNT_EV_UPPER,
                        MF_CNT_EV_PLATEAU, MF_CNT_EV_DEAD, MF_CNT_EV_FULL};
  const bool leader = (threadIdx.x & 31) == __ffs(mask) - 1;
#pragma unroll
  for (int k = 0; k < 6; k++) {
    const unsigned sum = __reduce_add_sync(mask, v[k]);
    if (leader && sum) atomicAdd(P.counters + cslot[k], (unsigned long long)sum);
  }
}

// A22 of each element from the row partials of G, summed in row order
template <int NQ1>
__global__ void __launch_bounds__(128) k_tri_u_a22(AsmParams P,
                                                   const double *gscr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.n_inner) return;
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  const int64_t m = P.inner[t];
  double Gt[NQ1];
#pragma unroll
  for (int q = 0; q < NQ1; q++) Gt[q] = 0.0;
  for (int p = 0; p <= 2 * P.R; p++) {
    const double *gp = gscr + ((int64_t)p * P.n_inner + t) * NQ1;
#pragma unroll
    for (int q = 0; q < NQ1; q++) Gt[q] += gp[q];
  }
  const double *c = M.elem_coords + m * M.nv_max * 2;
  const double e10 = xsub(c[2], c[0]), e11 = xsub(c[3], c[1]);
  const double e20 = xsub(c[4], c[0]), e21 = xsub(c[5], c[1]);
  const double sc = P.scale * (e10 * e21 - e11 * e20);
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const int64_t r = mdofs[i];
#pragma unroll
    for (int j = 0; j < 3; j++) {
      double b = 0.0;
#pragma unroll
      for (int q = 0; q < NQ1; q++)
        b = fma(Gt[q] * (Rr.tri_in_w[q] * Rr.phi_tri_in[q * 3 + i]),
                Rr.phi_tri_in[q * 3 + j], b);
      P.vals[pat_index(P.pat, r, mdofs[j])] += sc * b;
    }
  }
}

// ---- k_tri_q: k_tri_u with warp-cooperative full events ----
//
// Unstructured pairs take different Algorithm-1 paths, so the lanes of a
// k_tri_u warp diverge (ncu: ~6.6 of 32 threads active).  Here each lane
// walks its pair's tree (classification, dead events and the cheap plateau
// events inline) and only RECORDS its full L_max events as a bit mask over
// the 4^(L_max-1) <= 16 leaf sub-triangles.  The warp then integrates all
// recorded events of its 32 pairs together, 32 events per round, every
// lane running the identical 36/49-point-pair event code; each event's
// V contribution goes through shared memory back to its owner lane, which
// adds them in queue order (owner lane, then leaf index) -- deterministic.
// Requires eps > 0, shortcuts on and L_max <= 3 (else k_tri_u runs).
constexpr int kTriQWarps = 4;

// d = gy*NX + gx for a lattice id d < 2^24 (checked on the host): float
// quotient, then one exact integer correction step
MF_DEV void lattice_split(int d, int NX, float inv_nx, int &gx, int &gy) {
  gy = __float2int_rz(__int2float_rn(d) * inv_nx);
  gx = d - gy * NX;
  if (gx < 0) {
    gx += NX;
    gy--;
  } else if (gx >= NX) {
    gx -= NX;
    gy++;
  }
}

// blocks per SM of k_tri_q: 3 (168 registers) for large launches (R2
// 1.203 vs 1.209 s with 2); small, latency-bound launches run faster with
// 2 blocks of the 255-register build (R1 31.0 -> 26.4 ms, R2-small 220 ->
// 196 ms), so launch_tri_u picks by the launch's thread count
#ifndef MF_TRIQ_SMALL_THREADS
#define MF_TRIQ_SMALL_THREADS (148 * 384 * 4)
#endif

// Algorithm-1 decision for one sub-triangle at level L (shortcuts on):
// _kernels.py:224-251 plus the dead / plateau proofs at L_max
MF_DEV int tri_classify(const AsmParams &P, const double *g, int L,
                        const double *ilo, const double *ihi,
                        const double *pilo, const double *pihi, double fo) {
  double slo[2], shi[2];
  sub_bbox<1>(g, slo, shi);
  if (L < P.L_min) return ACT_SPLIT;
  if (L == P.L_max) {
    if (!(aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe)) return ACT_NONE;
    // dead / plateau proofs on the quadrature POINT sets (see mf_hex.cu
    // classify): the outer rule points lie in the sub-triangle shrunk
    // about its centroid by fo = 1 - 3 min(barycentric); pilo/pihi bound
    // the inner element's points.  Relative margins keep the proofs safe
    // under rounding; the event is counted either way.
    double qlo[2], qhi[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const double c = (g[k] + g[2 + k] + g[4 + k]) * (1.0 / 3.0);
      const double mg = 1e-9 * (shi[k] - slo[k]);
      qlo[k] = c + fo * (slo[k] - c) - mg;
      qhi[k] = c + fo * (shi[k] - c) + mg;
    }
    if (box_dead<2>(P, qlo, qhi, pilo, pihi)) return ACT_DEAD;
    if (aprx_max_sq<2>(qlo, qhi, pilo, pihi) < P.dm2 * (1.0 - 4e-9))
      return ACT_PLAT;
    return ACT_FULL;
  }
  if (aprx_max_lt_dme(P, aprx_max_sq<2>(slo, shi, ilo, ihi)))
    return ACT_UPPER;
  if (aprx_min_d<2>(slo, shi, ilo, ihi) < P.dpe) return ACT_SPLIT;
  return ACT_NONE;
}

MF_DEV void outer_map(const double *c, OuterTri &O) {
  const double e10 = c[2] - c[0], e11 = c[3] - c[1];
  const double e20 = c[4] - c[0], e21 = c[5] - c[1];
  const double idet = rcp_fast(e10 * e21 - e11 * e20);
  O.v0[0] = c[0];
  O.v0[1] = c[1];
  O.inv[0] = e21 * idet;
  O.inv[1] = -e20 * idet;
  O.inv[2] = -e11 * idet;
  O.inv[3] = e10 * idet;
}

template <int NQO, int NQ1, int MINB>
__global__ void __launch_bounds__(32 * kTriQWarps, MINB)
    k_tri_q(AsmParams P, int cls, double *gscr) {
  constexpr int NL = 3;
  constexpr int NV = NQ1 * NL;
  __shared__ double s_phiw[NQ1][NL];
  __shared__ double s_opts[2 * NQO], s_ow[NQO];
  // per-lane pair state, lane-major: inner points, outer root + inverse
  __shared__ double s_y[kTriQWarps][NQ1][2][32];
  __shared__ double s_root[kTriQWarps][6][32];   // outer root triangle
  // per-event V of a phase-B round; phase W reuses the first 11 rows for
  // the owners' inner boxes, plateau sums and point-set boxes
  constexpr int NRES = NV > 11 ? NV : 11;
  // (row pitch 33: the segment sums below read one ROW per lane)
  __shared__ double s_res[kTriQWarps][NRES][33];
  __shared__ int s_off[kTriQWarps][33];
  __shared__ unsigned s_mask[kTriQWarps][32];
  __shared__ int s_own[kTriQWarps][32];      // owner lane of a round's event
  // the lane's 3 pattern rows: rowptr base shifted to (ylo, xlo), width
  __shared__ long long s_rb[kTriQWarps][NL][32];
  __shared__ int s_wx[kTriQWarps][NL][32];
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * NL; i += blockDim.x) {
    const int q = i / NL, j = i % NL;
    s_phiw[q][j] = Rr.tri_in_w[q] * Rr.phi_tri_in[q * NL + j];
  }
  for (int i = threadIdx.x; i < NQO; i += blockDim.x) {
    s_opts[2 * i] = Rr.tri_out_pts[2 * i];
    s_opts[2 * i + 1] = Rr.tri_out_pts[2 * i + 1];
    s_ow[i] = Rr.tri_out_w[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < P.n_inner;
  const int Rs = P.R;
  const int pidx = cls + M.row_period * (int)blockIdx.y;  // dy + R
  const int dy = pidx - Rs;
  const int64_t m = valid ? P.inner[t] : P.inner[0];
  double G[NQ1];
#pragma unroll
  for (int q = 0; q < NQ1; q++) G[q] = 0.0;
  unsigned c_ev = 0, c_pairs = 0, c_up = 0, c_pl = 0, c_dead = 0, c_full = 0;
  const int cell = M.elem_cell[m];
  const int cx = cell % M.ncx, cy = cell / M.ncx;
  const int y2 = cy + dy;
  // candidate range of this lane's stencil row (empty for idle lanes)
  int64_t l = 0, l1 = 0;
  if (valid && y2 >= 0 && y2 < M.ncy) {
    l = M.cell_ptr[(int64_t)y2 * M.ncx + max(cx - Rs, 0)];
    l1 = M.cell_ptr[(int64_t)y2 * M.ncx + min(cx + Rs, M.ncx - 1) + 1];
  }
  double ilo[2], ihi[2], scale_in;
  ilo[0] = M.elem_lo[m * 2];
  ilo[1] = M.elem_lo[m * 2 + 1];
  ihi[0] = M.elem_hi[m * 2];
  ihi[1] = M.elem_hi[m * 2 + 1];
  {
    const double *c = M.elem_coords + m * M.nv_max * 2;
    const double e10 = xsub(c[2], c[0]), e11 = xsub(c[3], c[1]);
    const double e20 = xsub(c[4], c[0]), e21 = xsub(c[5], c[1]);
    scale_in = e10 * e21 - e11 * e20;
    for (int q = 0; q < NQ1; q++) {
      const double p0 = Rr.tri_in_pts[2 * q], p1 = Rr.tri_in_pts[2 * q + 1];
      s_y[w][q][0][lane] = xadd(xadd(c[0], xmul(p0, e10)), xmul(p1, e20));
      s_y[w][q][1][lane] = xadd(xadd(c[1], xmul(p0, e11)), xmul(p1, e21));
    }
  }
  // outer point shrink factor and the inner point-set box (proofs)
  double fo = 1.0;
  for (int q = 0; q < NQO; q++) {
    const double a = s_opts[2 * q], b = s_opts[2 * q + 1];
    fo = fmin(fo, fmin(fmin(a, b), 1.0 - a - b));
  }
  fo = fmin(1.0, 1.0 - 3.0 * fo + 1e-9);
  double pilo[2], pihi[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    double mn = 1e300, mx = -1e300;
    for (int q = 0; q < NQ1; q++) {
      mn = fmin(mn, s_y[w][q][k][lane]);
      mx = fmax(mx, s_y[w][q][k][lane]);
    }
    const double wd = ihi[k] - ilo[k];
    pilo[k] = mn - 1e-9 * wd;
    pihi[k] = mx + 1e-9 * wd;
  }
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
  const int NX = P.pat.NX, K = P.pat.K;
  const float inv_nx = 1.0f / (float)NX;
  // entry (r, c) = rowptr[r] + (gy_c - ylo) Wx + (gx_c - xlo)
  //             = rb + gy_c Wx + gx_c  with rb = rowptr[r] - ylo Wx - xlo
#pragma unroll
  for (int i = 0; i < NL; i++) {
    int rgx, rgy;
    lattice_split((int)mdofs[i], NX, inv_nx, rgx, rgy);
    const int xlo = max(rgx - K, 0);
    const int wx = min(rgx + K, NX - 1) - xlo + 1;
    s_rb[w][i][lane] = (long long)P.pat.rowptr[mdofs[i]] -
                       (long long)max(rgy - K, 0) * wx - xlo;
    s_wx[w][i][lane] = wx;
  }
  const int nleaf_bits = 2 * (P.L_max - 1);
  for (;;) {
    // ---- phase A: next candidate pair of this lane, walked alone ----
    bool have = false;
    while (l < l1) {
      if (P.outer_mask[l] && elem_gap<2>(M.elem_lo, M.elem_hi, l, m) < P.dpe) {
        have = true;
        break;
      }
      l++;
    }
    if (!__any_sync(0xffffffffu, have)) break;
    unsigned fmask = 0;
    unsigned ev = 0;
    double SP[NL] = {0.0, 0.0, 0.0};
    bool live = false;
    bool walk = false;
    if (have) {
      c_pairs++;
      const int64_t *ldofs = M.elem_dofs + l * M.nloc_max;
#pragma unroll
      for (int j = 0; j < NL; j++) {
        int gx, gy;
        lattice_split((int)ldofs[j], NX, inv_nx, gx, gy);
#pragma unroll
        for (int i = 0; i < NL; i++) {
          const int64_t sl = s_rb[w][i][lane] +
                             (int64_t)gy * s_wx[w][i][lane] + gx;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + sl));
        }
      }
      // root only; deeper levels are walked by the whole warp below
      double root[6];
      {
        const double *c = M.elem_coords + l * M.nv_max * 2;
#pragma unroll
        for (int u = 0; u < 6; u++) {
          root[u] = c[u];
          s_root[w][u][lane] = c[u];
        }
      }
      const int act = tri_classify(P, root, 1, ilo, ihi, pilo, pihi, fo);
      if (act >= ACT_UPPER) {
        ev++;
        if (act == ACT_UPPER) c_up++;
        if (act == ACT_DEAD) c_dead++;
        if (act == ACT_PLAT) c_pl++;
        if (act == ACT_FULL) {
          c_full++;
          fmask = 1u;
        }
        if (act == ACT_PLAT || act == ACT_UPPER) {
          live = true;
          OuterTri OT;
          outer_map(root, OT);
          tri_plateau<NQO>(P, root, OT, s_opts, s_ow, SP);
        }
      }
      walk = act == ACT_SPLIT;
    }
    // ---- phase W: the split pairs' sub-triangles, walked by the warp ----
    // A pair split at the root has 4^(L_max-1) <= 16 leaves; lane group g
    // (nper lanes) takes owner pair g of this round and lane s of the group
    // evaluates leaf s: its level-2 parent (the group's 4 lanes of one
    // parent agree on its class; lane k = 0 integrates a parent plateau
    // event), then the leaf itself.  Full leaves become the owner's fmask
    // bits, plateau contributions are reduced over the group (fixed
    // shuffle tree) and added to the owner's SP -- deterministic.
    unsigned wmask = __ballot_sync(0xffffffffu, walk);
    if (wmask) {
      const int nper = 1 << nleaf_bits;  // 4 (L_max 2) or 16 (L_max 3)
      const int grp = lane / nper, sl = lane % nper;
      double(*s_ib)[33] = s_res[w];         // owner inner boxes (4 rows)
      double(*s_sp)[33] = s_res[w] + 4;     // owner plateau sums (3 rows)
      double(*s_pb)[33] = s_res[w] + 7;     // owner point-set boxes (4)
      s_ib[0][lane] = ilo[0];
      s_ib[1][lane] = ilo[1];
      s_ib[2][lane] = ihi[0];
      s_ib[3][lane] = ihi[1];
      s_pb[0][lane] = pilo[0];
      s_pb[1][lane] = pilo[1];
      s_pb[2][lane] = pihi[0];
      s_pb[3][lane] = pihi[1];
      __syncwarp();
      while (wmask) {
        const int cnt = __popc(wmask);
        const int o = grp < cnt ? nth_set_bit(wmask, grp + 1) : -1;
        double spi[NL] = {0.0, 0.0, 0.0};
        bool fl = false, lv = false;
        if (o >= 0) {
          double rt[6], blo[2], bhi[2];
#pragma unroll
          for (int u = 0; u < 6; u++) rt[u] = s_root[w][u][o];
          blo[0] = s_ib[0][o];
          blo[1] = s_ib[1][o];
          bhi[0] = s_ib[2][o];
          bhi[1] = s_ib[3][o];
          double qlo[2], qhi[2];
          qlo[0] = s_pb[0][o];
          qlo[1] = s_pb[1][o];
          qhi[0] = s_pb[2][o];
          qhi[1] = s_pb[3][o];
          OuterTri O;
          outer_map(rt, O);
          double g2[6];
          make_child<1>(rt, nleaf_bits == 2 ? sl : (sl >> 2), g2);
          int a = tri_classify(P, g2, 2, blo, bhi, qlo, qhi, fo);
          if (nleaf_bits == 4) {
            if (a == ACT_UPPER) {
              if ((sl & 3) == 0) {
                c_ev++;
                c_up++;
                lv = true;
                tri_plateau<NQO>(P, g2, O, s_opts, s_ow, spi);
              }
              a = ACT_NONE;
            } else if (a == ACT_SPLIT) {
              double g3[6];
              make_child<1>(g2, sl & 3, g3);
#pragma unroll
              for (int u = 0; u < 6; u++) g2[u] = g3[u];
              a = tri_classify(P, g2, 3, blo, bhi, qlo, qhi, fo);
            } else {
              a = ACT_NONE;
            }
          }
          // a: the leaf's class at L_max (or ACT_NONE)
          if (a >= ACT_UPPER) {
            c_ev++;
            if (a == ACT_DEAD) c_dead++;
            if (a == ACT_PLAT) {
              c_pl++;
              lv = true;
              tri_plateau<NQO>(P, g2, O, s_opts, s_ow, spi);
            }
            if (a == ACT_FULL) {
              c_full++;
              fl = true;
            }
          }
        }
        const unsigned fb = __ballot_sync(0xffffffffu, fl);
        const unsigned lb = __ballot_sync(0xffffffffu, fl || lv);
        for (int d = nper >> 1; d >= 1; d >>= 1)
#pragma unroll
          for (int k = 0; k < NL; k++)
            spi[k] += __shfl_xor_sync(0xffffffffu, spi[k], d);
        if (o >= 0 && sl == 0) {
          const unsigned gm = (1u << nper) - 1u;
          const unsigned fg = (fb >> (grp * nper)) & gm;
          const unsigned lg = (lb >> (grp * nper)) & gm;
          s_mask[w][o] = fg | (lg ? 0x80000000u : 0u);
#pragma unroll
          for (int k = 0; k < NL; k++) s_sp[k][o] = spi[k];
        }
        for (int k = 0; k < 32 / nper && wmask; k++) wmask &= wmask - 1;
      }
      __syncwarp();
      if (walk) {
        const unsigned v = s_mask[w][lane];
        fmask = v & 0xffffu;
        live |= (v >> 31) != 0u;
#pragma unroll
        for (int k = 0; k < NL; k++) SP[k] += s_sp[k][lane];
      }
      __syncwarp();
    }
    if (have) {
      live |= fmask != 0;
    }
    // ---- phase B: the warp's full events, 32 per round, converged ----
    const int cnt = __popc(fmask);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;  // exclusive prefix
    s_off[w][lane] = off;
    s_mask[w][lane] = fmask;
    if (lane == 31) s_off[w][32] = total;
    __syncwarp();
    double V[NQ1][NL];
#pragma unroll
    for (int q = 0; q < NQ1; q++)
#pragma unroll
      for (int j = 0; j < NL; j++) V[q][j] = 0.0;
    for (int base = 0; base < total; base += 32) {
      const int g = base + lane;
      if (g < total) {
        // owner lane o: s_off[w][o] <= g < s_off[w][o + 1]
        int o = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1)
          if (s_off[w][o + step] <= g) o += step;
        const unsigned om = s_mask[w][o];
        const int leaf = nth_set_bit(om, g - s_off[w][o] + 1);
        double gg[6];
#pragma unroll
        for (int u = 0; u < 6; u++) gg[u] = s_root[w][u][o];
        // the owner's outer inverse map, recomputed from its root exactly
        // as in phase A
        OuterTri O;
        {
          const double e10 = gg[2] - gg[0], e11 = gg[3] - gg[1];
          const double e20 = gg[4] - gg[0], e21 = gg[5] - gg[1];
          const double idet = rcp_fast(e10 * e21 - e11 * e20);
          O.v0[0] = gg[0];
          O.v0[1] = gg[1];
          O.inv[0] = e21 * idet;
          O.inv[1] = -e20 * idet;
          O.inv[2] = -e11 * idet;
          O.inv[3] = e10 * idet;
        }
        for (int b = nleaf_bits - 2; b >= 0; b -= 2) {
          double c[6];
          make_child<1>(gg, (leaf >> b) & 3, c);
#pragma unroll
          for (int u = 0; u < 6; u++) gg[u] = c[u];
        }
        double yy[NQ1][2];
#pragma unroll
        for (int q = 0; q < NQ1; q++) {
          yy[q][0] = s_y[w][q][0][o];
          yy[q][1] = s_y[w][q][1][o];
        }
        double Ve[NQ1][NL];
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
          for (int j = 0; j < NL; j++) Ve[q][j] = 0.0;
        tri_full<NQO, NQ1, false, false>(P, gg, O, yy, s_opts, s_ow, Ve);
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
          for (int j = 0; j < NL; j++) s_res[w][q * NL + j][lane] = Ve[q][j];
        s_own[w][lane] = o;
      }
      __syncwarp();
      // Segment sums: lane v < NV walks row v of the round's results and
      // sums each owner's run of events in queue order, leaving the sum in
      // the run's first column; then every owner adds ONE value per row.
      // (Each owner used to walk its own events: the warp then ran the
      // longest owner's loop with 2 NV instructions per event -- 12% of
      // the kernel's instructions.)  Fixed order: deterministic.
      const int nround = min(32, total - base);
      if (lane < NV) {
        double *row = s_res[w][lane];
        int cur = s_own[w][0], first = 0;
        double acc = row[0];
        for (int k = 1; k < nround; k++) {
          const int ok = s_own[w][k];
          const double v = row[k];
          if (ok != cur) {
            row[first] = acc;
            acc = 0.0;
            cur = ok;
            first = k;
          }
          acc += v;
        }
        row[first] = acc;
      }
      __syncwarp();
      const int a = max(off, base), b = min(off + cnt, base + 32);
      if (a < b) {
#pragma unroll
        for (int q = 0; q < NQ1; q++)
#pragma unroll
          for (int j = 0; j < NL; j++) V[q][j] += s_res[w][q * NL + j][a - base];
      }
      __syncwarp();
    }
    if (have) {
      c_ev += ev;
      // dead-only pairs add an exactly zero block: skipped
      if (live) {
        const int64_t *ldofs = M.elem_dofs + l * M.nloc_max;
        const double spsum = (SP[0] + SP[1]) + SP[2];
        const double sc = -P.scale * scale_in;
        int cgx[NL], cgy[NL];
#pragma unroll
        for (int j = 0; j < NL; j++)
          lattice_split((int)ldofs[j], NX, inv_nx, cgx[j], cgy[j]);
        double old[NL][NL];
#pragma unroll
        for (int i = 0; i < NL; i++)
#pragma unroll
          for (int j = 0; j < NL; j++)
            old[i][j] = P.vals[s_rb[w][i][lane] +
                               (int64_t)cgy[j] * s_wx[w][i][lane] + cgx[j]];
#pragma unroll
        for (int i = 0; i < NL; i++) {
          const int64_t rb = s_rb[w][i][lane];
          const int wx = s_wx[w][i][lane];
          double mi = 0.0;
#pragma unroll
          for (int q = 0; q < NQ1; q++) mi += s_phiw[q][i];
#pragma unroll
          for (int j = 0; j < NL; j++) {
            double bsum = mi * SP[j];
#pragma unroll
            for (int q = 0; q < NQ1; q++)
              bsum = fma(s_phiw[q][i], V[q][j], bsum);
            P.vals[rb + (int64_t)cgy[j] * wx + cgx[j]] = old[i][j] + sc * bsum;
          }
        }
#pragma unroll
        for (int q = 0; q < NQ1; q++) {
          double sg = spsum;
#pragma unroll
          for (int j = 0; j < NL; j++) sg += V[q][j];
          G[q] += sg;
        }
      }
      l++;
    }
  }
  if (valid) {
    double *gp = gscr + ((int64_t)pidx * P.n_inner + t) * NQ1;
#pragma unroll
    for (int q = 0; q < NQ1; q++) gp[q] = G[q];
  }
  const unsigned v[6] = {c_ev, c_pairs, c_up, c_pl, c_dead, c_full};
  const int cslot[6] = {MF_CNT_EVENTS, MF_CNT_PAIRS, MF_CNT_EV_UPPER,
                        MF_CNT_EV_PLATEAU, MF_CNT_EV_DEAD, MF_CNT_EV_FULL};
#pragma unroll
  for (int k = 0; k < 6; k++) {
    const unsigned sum = __reduce_add_sync(0xffffffffu, v[k]);
    if (lane == 0 && sum) atomicAdd(P.counters + cslot[k], (unsigned long long)sum);
  }
}

template <int NQO, int NQ1>
cudaError_t launch_tri_u(const AsmParams &P, double *gscr, cudaStream_t s) {
  const unsigned gx = (unsigned)((P.n_inner + 127) / 128);
  const int per = P.mesh.row_period, rows = 2 * P.R + 1;
  const bool queue = MF_TRI_QUEUE && P.eps > 0.0 && P.shortcuts &&
                     P.L_max <= 3;
  for (int cls = 0; cls < per; cls++) {
    const int n = (rows - cls + per - 1) / per;
    if (n < 1) continue;
    if (queue && (int64_t)P.n_inner * n < MF_TRIQ_SMALL_THREADS)
      k_tri_q<NQO, NQ1, 2><<<dim3(gx, n), 32 * kTriQWarps, 0, s>>>(P, cls,
                                                                 gscr);
    else if (queue)
      k_tri_q<NQO, NQ1, 3><<<dim3(gx, n), 32 * kTriQWarps, 0, s>>>(P, cls,
                                                                 gscr);
    else
      k_tri_u<NQO, NQ1><<<dim3(gx, n), 128, 0, s>>>(P, cls, gscr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_tri_u_a22<NQ1><<<gx, 128, 0, s>>>(P, gscr);
  return cudaGetLastError();
}

template <int KIND, int NO, int NI>
cudaError_t launch(const AsmParams &P, cudaStream_t s) {
  const int block = 128;
  const int64_t grid = (P.n_inner + block - 1) / block;
  k_2d<KIND, NO, NI><<<(unsigned)grid, block, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace

bool mf_2d_supported(const AsmParams &P) {
  const MfMesh &M = P.mesh;
  if (M.dim != 2 || M.degree != 1 || P.L_max > kMaxLevels) return false;
  if (M.layout != 0) return false;  // unstructured: k_tri_u
  const MfRules &R = P.rules;
  if (M.kinds_present == 2) {  // pure triangle mesh
    return M.nloc_max == 3 && R.nq_tri_out == 7 && R.nq_tri_in == 7;
  }
  if (M.kinds_present != 1) return false;  // mixed -> generic kernel
  if (R.n1d_box_in < 1 || R.n1d_box_in > 3) return false;
  if (R.n1d_box_out < 1 || R.n1d_box_out > 4) return false;
  return R.nq_box_in == R.n1d_box_in * R.n1d_box_in &&
         R.nq_box_out == R.n1d_box_out * R.n1d_box_out;
}

cudaError_t mf_launch_2d(const AsmParams &P, cudaStream_t s) {
  if (P.mesh.kinds_present == 2) return launch<1, 7, 7>(P, s);
  const int no = P.rules.n1d_box_out, ni = P.rules.n1d_box_in;
#define MF_Q(NO_, NI_) \
  if (no == NO_ && ni == NI_) return launch<0, NO_, NI_>(P, s);
  MF_Q(1, 1) MF_Q(2, 1) MF_Q(3, 1) MF_Q(4, 1)
  MF_Q(1, 2) MF_Q(2, 2) MF_Q(3, 2) MF_Q(4, 2)
  MF_Q(1, 3) MF_Q(2, 3) MF_Q(3, 3) MF_Q(4, 3)
#undef MF_Q
  return cudaErrorNotSupported;
}

bool mf_tri_u_supported(const AsmParams &P) {
  const MfMesh &M = P.mesh;
  if (M.layout != 1 || M.dim != 2 || M.degree != 1 || M.kinds_present != 2)
    return false;
  if (M.nloc_max != 3 || M.row_period < 2 || P.L_max > kMaxLevels)
    return false;
  if (P.pat.n >= (1 << 24)) return false;  // lattice_split range
  const int no = P.rules.nq_tri_out, ni = P.rules.nq_tri_in;
  return (no == 3 || no == 6 || no == 7) && (ni == 3 || ni == 6 || ni == 7);
}

size_t mf_tri_u_scratch_doubles(const AsmParams &P, int64_t n_colour_max) {
  return (size_t)(2 * P.R + 1) * (size_t)n_colour_max *
         (size_t)P.rules.nq_tri_in;
}

cudaError_t mf_launch_tri_u(const AsmParams &P, double *gscr,
                            cudaStream_t s) {
  const int no = P.rules.nq_tri_out, ni = P.rules.nq_tri_in;
#define MF_TU(NO_, NI_) \
  if (no == NO_ && ni == NI_) return launch_tri_u<NO_, NI_>(P, gscr, s);
  MF_TU(3, 3) MF_TU(3, 6) MF_TU(3, 7)
  MF_TU(6, 3) MF_TU(6, 6) MF_TU(6, 7)
  MF_TU(7, 3) MF_TU(7, 6) MF_TU(7, 7)
#undef MF_TU
  return cudaErrorNotSupported;
}
