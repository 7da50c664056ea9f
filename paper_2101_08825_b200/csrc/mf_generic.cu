// mf_generic.cu -- generic adaptive pair assembly (all kinds/degrees/rules).
//
// One thread per INNER element m of the current colour.  The thread
// enumerates its outer partners l in the (2R+1)^dim cell stencil with the
// exact candidate test (max-axis gap < delta+eps, _kernels.py:1225-1233; the
// relation is symmetric so this is the transpose of the reference's
// J_l lists), runs Algorithm 1 per pair (_pair_blocks, _kernels.py:184-313)
// as a depth-first walk that keeps one geometry per level, integrates each
// event in the reference's rank-1 form (_event_box/_event_tri,
// _kernels.py:105-181) and adds the inner-row blocks into vals.  A22 is
// folded once per inner element from the element-level sum of gsum over all
// its pairs (the reference folds per pair, _kernels.py:303-312; same sum).
//
// All of a pair's entries lie in rows of the inner element
// (_kernels.py:483-486), and same-colour elements share no DOF, so the
// launch is race-free without atomics and deterministic.
//
// This kernel is the fallback for configurations the specialised kernels
// (mf_hex.cu, mf_tri.cu) do not cover: mixed meshes, degree 2, large rules,
// deep L_max.
#include "mf_common.cuh"

namespace {

constexpr int kLevels = 25;  // L_max <= 24 (assembly.py:65)

struct Outer {
  int kind;       // 0 quad, 1 tri, 2 hex
  int nloc;
  double geo[6];  // box lo/hi or tri vertices
  double lo[3], hi[3];
  double v0[2], inv[4];
};

template <int DIM>
MF_DEV void sub_bbox(int kind, const double *g, double *slo, double *shi) {
  if (kind == 1) {
    slo[0] = pmin(g[0], pmin(g[2], g[4]));
    shi[0] = pmax(g[0], pmax(g[2], g[4]));
    slo[1] = pmin(g[1], pmin(g[3], g[5]));
    shi[1] = pmax(g[1], pmax(g[3], g[5]));
  } else {
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      slo[k] = g[k];
      shi[k] = g[DIM + k];
    }
  }
}

// child b of sub-cell g (_kernels.py:253-302), exact midpoint arithmetic
template <int DIM>
MF_DEV void make_child(int kind, const double *g, int b, double *c) {
  if (kind == 1) {
    double m010 = xmul(0.5, xadd(g[0], g[2]));
    double m011 = xmul(0.5, xadd(g[1], g[3]));
    double m120 = xmul(0.5, xadd(g[2], g[4]));
    double m121 = xmul(0.5, xadd(g[3], g[5]));
    double m200 = xmul(0.5, xadd(g[4], g[0]));
    double m201 = xmul(0.5, xadd(g[5], g[1]));
    if (b == 0) {
      c[0] = g[0]; c[1] = g[1]; c[2] = m010; c[3] = m011; c[4] = m200;
      c[5] = m201;
    } else if (b == 1) {
      c[0] = m010; c[1] = m011; c[2] = g[2]; c[3] = g[3]; c[4] = m120;
      c[5] = m121;
    } else if (b == 2) {
      c[0] = m200; c[1] = m201; c[2] = m120; c[3] = m121; c[4] = g[4];
      c[5] = g[5];
    } else {
      c[0] = m010; c[1] = m011; c[2] = m120; c[3] = m121; c[4] = m200;
      c[5] = m201;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    double lo = g[k], hi = g[DIM + k];
    double mid = xmul(0.5, xadd(lo, hi));
    if (((b >> k) & 1) == 0) {
      c[k] = lo;
      c[DIM + k] = mid;
    } else {
      c[k] = mid;
      c[DIM + k] = hi;
    }
  }
}

struct Inner {
  int kind, nq, nloc;
  const double *pts, *w, *phi;
  double lo[3], hi[3];
  double c0[2], e1[2], e2[2];  // tri: vertex 0 and edges
  double scale_w;              // det (tri) or jac (box)
};

// physical inner point q (_inner_data, _kernels.py:316-340), exact
template <int DIM>
MF_DEV void inner_point(const Inner &I, int q, double *y) {
  if (I.kind == 1) {
    double p0 = I.pts[q * 2], p1 = I.pts[q * 2 + 1];
    y[0] = xadd(xadd(I.c0[0], xmul(p0, I.e1[0])), xmul(p1, I.e2[0]));
    y[1] = xadd(xadd(I.c0[1], xmul(p0, I.e1[1])), xmul(p1, I.e2[1]));
    return;
  }
#pragma unroll
  for (int k = 0; k < DIM; k++)
    y[k] = xadd(I.lo[k], xmul(xmul(xadd(I.pts[q * DIM + k], 1.0), 0.5),
                              xsub(I.hi[k], I.lo[k])));
}

// one integration event on sub-cell g (reference rank-1 form)
template <int DIM, int NLM>
MF_DEV void event_full(const AsmParams &P, const Outer &O, const double *g,
                       const Inner &I, double *b21, double *G) {
  const MfRules &Rr = P.rules;
  int degree = P.mesh.degree;
  double phi2[NLM];
  if (O.kind == 1) {
    double e10 = xsub(g[2], g[0]), e11 = xsub(g[3], g[1]);
    double e20 = xsub(g[4], g[0]), e21 = xsub(g[5], g[1]);
    double det = e10 * e21 - e11 * e20;
    for (int q2 = 0; q2 < Rr.nq_tri_out; q2++) {
      double px = Rr.tri_out_pts[q2 * 2], py = Rr.tri_out_pts[q2 * 2 + 1];
      double x[3];
      x[0] = xadd(xadd(g[0], xmul(px, e10)), xmul(py, e20));
      x[1] = xadd(xadd(g[1], xmul(px, e11)), xmul(py, e21));
      double w2q = Rr.tri_out_w[q2] * det * P.cde * (1.0 / 256.0);
      double dx0 = x[0] - O.v0[0], dx1 = x[1] - O.v0[1];
      double rx = O.inv[0] * dx0 + O.inv[1] * dx1;
      double ry = O.inv[2] * dx0 + O.inv[3] * dx1;
      shape_at(1, degree, 2, rx, ry, 0.0, phi2);
      for (int q1 = 0; q1 < I.nq; q1++) {
        double y[3];
        inner_point<DIM>(I, q1, y);
        double dx = xsub(x[0], y[0]), dy = xsub(x[1], y[1]);
        double d2 = xadd(xmul(dx, dx), xmul(dy, dy));
        if (d2 >= P.dp2) continue;
        double tq = mu256(P, d2) * w2q;
        G[q1] += tq;
        double tw = tq * I.w[q1] * I.scale_w;
        for (int i = 0; i < I.nloc; i++) {
          double ci = tw * I.phi[q1 * I.nloc + i];
          for (int j = 0; j < O.nloc; j++) b21[i * NLM + j] -= ci * phi2[j];
        }
      }
    }
    return;
  }
  double jac = 1.0;
#pragma unroll
  for (int k = 0; k < DIM; k++) jac *= 0.5 * (g[DIM + k] - g[k]);
  for (int q2 = 0; q2 < Rr.nq_box_out; q2++) {
    double x[3], r[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      x[k] = xadd(g[k], xmul(xmul(xadd(Rr.box_out_pts[q2 * DIM + k], 1.0),
                                  0.5),
                             xsub(g[DIM + k], g[k])));
      r[k] = (x[k] - O.lo[k]) / (O.hi[k] - O.lo[k]) * 2.0 - 1.0;
    }
    double w2q = Rr.box_out_w[q2] * jac * P.cde * (1.0 / 256.0);
    shape_at(O.kind, degree, DIM, r[0], r[1], r[2], phi2);
    for (int q1 = 0; q1 < I.nq; q1++) {
      double y[3];
      inner_point<DIM>(I, q1, y);
      double d2 = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; k++) {
        double dk = xsub(x[k], y[k]);
        d2 = (k == 0) ? xmul(dk, dk) : xadd(d2, xmul(dk, dk));
      }
      if (d2 >= P.dp2) continue;
      double tq = mu256(P, d2) * w2q;
      G[q1] += tq;
      double tw = tq * I.w[q1] * I.scale_w;
      for (int i = 0; i < I.nloc; i++) {
        double ci = tw * I.phi[q1 * I.nloc + i];
        for (int j = 0; j < O.nloc; j++) b21[i * NLM + j] -= ci * phi2[j];
      }
    }
  }
}

// plateau shortcut: every point pair has mu == 1 (sub-cell proven inside
// delta-eps), so the event is rank-1:  b21 -= cde * m (x) S,  G += cde * W
template <int DIM, int NLM>
MF_DEV void event_plateau(const AsmParams &P, const Outer &O, const double *g,
                          const Inner &I, const double *mvec, double *b21,
                          double &Gall) {
  const MfRules &Rr = P.rules;
  int degree = P.mesh.degree;
  double phi2[NLM], S[NLM];
  for (int j = 0; j < O.nloc; j++) S[j] = 0.0;
  double W = 0.0;
  if (O.kind == 1) {
    double e10 = g[2] - g[0], e11 = g[3] - g[1];
    double e20 = g[4] - g[0], e21 = g[5] - g[1];
    double det = e10 * e21 - e11 * e20;
    for (int q2 = 0; q2 < Rr.nq_tri_out; q2++) {
      double px = Rr.tri_out_pts[q2 * 2], py = Rr.tri_out_pts[q2 * 2 + 1];
      double x0 = g[0] + px * e10 + py * e20;
      double x1 = g[1] + px * e11 + py * e21;
      double w2q = Rr.tri_out_w[q2] * det;
      double dx0 = x0 - O.v0[0], dx1 = x1 - O.v0[1];
      shape_at(1, degree, 2, O.inv[0] * dx0 + O.inv[1] * dx1,
               O.inv[2] * dx0 + O.inv[3] * dx1, 0.0, phi2);
      W += w2q;
      for (int j = 0; j < O.nloc; j++) S[j] += w2q * phi2[j];
    }
  } else {
    double jac = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; k++) jac *= 0.5 * (g[DIM + k] - g[k]);
    for (int q2 = 0; q2 < Rr.nq_box_out; q2++) {
      double r[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < DIM; k++) {
        double x = g[k] + (Rr.box_out_pts[q2 * DIM + k] + 1.0) * 0.5 *
                              (g[DIM + k] - g[k]);
        r[k] = (x - O.lo[k]) / (O.hi[k] - O.lo[k]) * 2.0 - 1.0;
      }
      double w2q = Rr.box_out_w[q2] * jac;
      shape_at(O.kind, degree, DIM, r[0], r[1], r[2], phi2);
      W += w2q;
      for (int j = 0; j < O.nloc; j++) S[j] += w2q * phi2[j];
    }
  }
  Gall += P.cde * W;
  for (int i = 0; i < I.nloc; i++) {
    double ci = P.cde * mvec[i];
    for (int j = 0; j < O.nloc; j++) b21[i * NLM + j] -= ci * S[j];
  }
}

// Algorithm 1 for one (outer O, inner I) pair (_pair_blocks,
// _kernels.py:184-313): depth-first walk with one geometry per level and
// the reference's midpoint arithmetic.  Adds the A21 block into b21, the
// per-q1 gamma sums into G (plus the q1-independent plateau part into
// Gall) and returns the event count.
struct EvCounts {
  unsigned long long up, pl, dead, full;
};

template <int DIM, int NLM>
MF_DEV unsigned long long pair_run(const AsmParams &P, const Outer &O,
                                   const Inner &I, const double *mvec,
                                   double *b21, double *G, double &Gall,
                                   EvCounts &cnt) {
  const int nchild = O.kind == 1 ? 4 : (1 << DIM);
  double geo[kLevels + 1][6];
  int child[kLevels + 1];
  for (int u = 0; u < 6; u++) geo[1][u] = O.geo[u];
  int L = 1;
  unsigned long long ev = 0;
  for (;;) {
    double slo[3], shi[3];
    sub_bbox<DIM>(O.kind, geo[L], slo, shi);
    bool split = false, integ = false;
    if (L < P.L_min) {
      split = true;
    } else if (L == P.L_max) {
      integ = aprx_min_d<DIM>(slo, shi, I.lo, I.hi) < P.dpe;
    } else if (aprx_max_lt_dme(P, aprx_max_sq<DIM>(slo, shi, I.lo, I.hi))) {
      integ = true;
    } else if (aprx_min_d<DIM>(slo, shi, I.lo, I.hi) < P.dpe) {
      split = true;
    }
    if (integ) {
      ev++;
      if (L < P.L_max) {
        cnt.up++;
        if (P.shortcuts)
          event_plateau<DIM, NLM>(P, O, geo[L], I, mvec, b21, Gall);
        else
          event_full<DIM, NLM>(P, O, geo[L], I, b21, G);
      } else if (P.shortcuts && box_dead<DIM>(P, slo, shi, I.lo, I.hi)) {
        cnt.dead++;
      } else if (P.shortcuts &&
                 aprx_max_lt_dme(P, aprx_max_sq<DIM>(slo, shi, I.lo, I.hi))) {
        cnt.pl++;
        event_plateau<DIM, NLM>(P, O, geo[L], I, mvec, b21, Gall);
      } else {
        cnt.full++;
        event_full<DIM, NLM>(P, O, geo[L], I, b21, G);
      }
    }
    if (split) {
      ++L;
      child[L] = 0;
      make_child<DIM>(O.kind, geo[L - 1], 0, geo[L]);
      continue;
    }
    bool done = false;
    for (;;) {
      if (L == 1) {
        done = true;
        break;
      }
      if (++child[L] < nchild) {
        make_child<DIM>(O.kind, geo[L - 1], child[L], geo[L]);
        break;
      }
      --L;
    }
    if (done) break;
  }
  return ev;
}

MF_DEV void scatter_add(const AsmParams &P, const int64_t *rows, int nr,
                        const int64_t *cols, int nc, const double *blk,
                        int ld) {
  for (int i = 0; i < nr; i++) {
    int64_t r = rows[i];
    for (int j = 0; j < nc; j++) {
      int64_t idx = pat_index(P.pat, r, cols[j]);
      P.vals[idx] += P.scale * blk[i * ld + j];
    }
  }
}

template <int DIM, int NLM>
__global__ void __launch_bounds__(128)
    k_generic(AsmParams P) {
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  double *G = P.scratch + tid * P.scratch_stride;
  unsigned long long c_ev = 0, c_pairs = 0;
  EvCounts cnt = {0, 0, 0, 0};
  for (int64_t t = tid; t < P.n_inner; t += nthreads) {
    const int64_t m = P.inner[t];
    Inner I;
    I.kind = M.elem_kind[m];
    const bool itri = I.kind == 1;
    I.nq = itri ? Rr.nq_tri_in : Rr.nq_box_in;
    I.nloc = itri ? P.nl_tri : P.nl_box;
    I.pts = itri ? Rr.tri_in_pts : Rr.box_in_pts;
    I.w = itri ? Rr.tri_in_w : Rr.box_in_w;
    I.phi = itri ? Rr.phi_tri_in : Rr.phi_box_in;
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      I.lo[k] = M.elem_lo[m * DIM + k];
      I.hi[k] = M.elem_hi[m * DIM + k];
    }
    if (itri) {
      const double *c = M.elem_coords + (size_t)m * M.nv_max * DIM;
      I.c0[0] = c[0];
      I.c0[1] = c[1];
      I.e1[0] = xsub(c[DIM], c[0]);
      I.e1[1] = xsub(c[DIM + 1], c[1]);
      I.e2[0] = xsub(c[2 * DIM], c[0]);
      I.e2[1] = xsub(c[2 * DIM + 1], c[1]);
      I.scale_w = I.e1[0] * I.e2[1] - I.e1[1] * I.e2[0];
    } else {
      double jac = 1.0;
#pragma unroll
      for (int k = 0; k < DIM; k++) jac *= 0.5 * (I.hi[k] - I.lo[k]);
      I.scale_w = jac;
    }
    // m_i = int phi_i over the inner element (plateau shortcut)
    double mvec[NLM];
    for (int i = 0; i < I.nloc; i++) {
      double s = 0.0;
      for (int q = 0; q < I.nq; q++) s += I.w[q] * I.phi[q * I.nloc + i];
      mvec[i] = s * I.scale_w;
    }
    for (int q = 0; q < I.nq; q++) G[q] = 0.0;
    double Gall = 0.0;  // plateau contributions common to every q1
    const int64_t *mdofs = M.elem_dofs + (size_t)m * M.nloc_max;
    // pair source: the explicit list of mf_general_core_lists (every
    // listed pair runs, as _general_core does, _kernels.py:432-438), or
    // the cell stencil filtered by the outer mask and the box gap
    const bool listed = P.list_begin != nullptr;
    int cx = 0, cy = 0, cz = 0;
    if (!listed) cell_coords(M.elem_cell[m], M.ncx, M.ncy, cx, cy, cz);
    const int R = listed ? 0 : P.R;
    const int zlo = DIM == 3 && !listed ? max(cz - R, 0) : 0;
    const int zhi = DIM == 3 && !listed ? min(cz + R, M.ncz - 1) : 0;
    const int yhi = listed ? 0 : min(cy + R, M.ncy - 1);
    const int xhi = listed ? 0 : min(cx + R, M.ncx - 1);
    for (int z2 = zlo; z2 <= zhi; z2++)
      for (int y2 = listed ? 0 : max(cy - R, 0); y2 <= yhi; y2++)
        for (int x2 = listed ? 0 : max(cx - R, 0); x2 <= xhi; x2++) {
          int64_t k0, k1;
          if (listed) {
            k0 = P.list_begin[t];
            k1 = P.list_end[t];
          } else {
            const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
            k0 = M.cell_ptr[c2];
            k1 = M.cell_ptr[c2 + 1];
          }
          for (int64_t k = k0; k < k1; k++) {
            const int64_t l = listed ? P.list_outer[k] : k;
            if (!listed) {
              if (!P.outer_mask[l]) continue;
              if (!(elem_gap<DIM>(M.elem_lo, M.elem_hi, l, m) < P.dpe))
                continue;
            }
            c_pairs++;
            Outer O;
            O.kind = M.elem_kind[l];
            O.nloc = O.kind == 1 ? P.nl_tri : P.nl_box;
            const double *lc = M.elem_coords + (size_t)l * M.nv_max * DIM;
            if (O.kind == 1) {
              for (int v = 0; v < 3; v++) {
                O.geo[2 * v] = lc[v * DIM];
                O.geo[2 * v + 1] = lc[v * DIM + 1];
              }
              double e10 = lc[DIM] - lc[0], e11 = lc[DIM + 1] - lc[1];
              double e20 = lc[2 * DIM] - lc[0], e21 = lc[2 * DIM + 1] - lc[1];
              double det = e10 * e21 - e11 * e20;
              O.v0[0] = lc[0];
              O.v0[1] = lc[1];
              O.inv[0] = e21 / det;
              O.inv[1] = -e20 / det;
              O.inv[2] = -e11 / det;
              O.inv[3] = e10 / det;
            } else {
#pragma unroll
              for (int k = 0; k < DIM; k++) {
                O.lo[k] = M.elem_lo[l * DIM + k];
                O.hi[k] = M.elem_hi[l * DIM + k];
                O.geo[k] = O.lo[k];
                O.geo[DIM + k] = O.hi[k];
              }
            }
            double b21[NLM * NLM];
            for (int i = 0; i < I.nloc * NLM; i++) b21[i] = 0.0;
            const unsigned long long ev =
                pair_run<DIM, NLM>(P, O, I, mvec, b21, G, Gall, cnt);
            if (ev) {
              c_ev += ev;
              scatter_add(P, mdofs, I.nloc, M.elem_dofs + (size_t)l * M.nloc_max,
                          O.nloc, b21, NLM);
            }
          }
        }
    // A22 for the whole element: sum_q1 G[q1] w1[q1] PHI1 PHI1^T
    double b22[NLM * NLM];
    for (int i = 0; i < I.nloc * NLM; i++) b22[i] = 0.0;
    bool any = Gall != 0.0;
    for (int q = 0; q < I.nq; q++) {
      double s = (G[q] + Gall) * I.w[q] * I.scale_w;
      if (s == 0.0) continue;
      any = true;
      for (int i = 0; i < I.nloc; i++) {
        double ci = s * I.phi[q * I.nloc + i];
        for (int j = 0; j < I.nloc; j++)
          b22[i * NLM + j] += ci * I.phi[q * I.nloc + j];
      }
    }
    if (any) scatter_add(P, mdofs, I.nloc, mdofs, I.nloc, b22, NLM);
  }
  unsigned long long *C = P.counters;
  counter_add(C + MF_CNT_EVENTS, c_ev);
  counter_add(C + MF_CNT_PAIRS, c_pairs);
  counter_add(C + MF_CNT_EV_UPPER, cnt.up);
  counter_add(C + MF_CNT_EV_PLATEAU, cnt.pl);
  counter_add(C + MF_CNT_EV_DEAD, cnt.dead);
  counter_add(C + MF_CNT_EV_FULL, cnt.full);
}

}  // namespace

// launch helper used by mf_capi.cu
cudaError_t mf_launch_generic(const AsmParams &P, int grid, int block,
                              cudaStream_t s) {
  int dim = P.mesh.dim;
  int nlm = P.nl_box > P.nl_tri ? P.nl_box : P.nl_tri;
  if (dim == 2) {
    if (nlm <= 9)
      k_generic<2, 9><<<grid, block, 0, s>>>(P);
    else
      return cudaErrorInvalidValue;
  } else {
    if (nlm <= 8)
      k_generic<3, 8><<<grid, block, 0, s>>>(P);
    else if (nlm <= 27)
      k_generic<3, 27><<<grid, block, 0, s>>>(P);
    else
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ===========================================================================
// Offset-blocked strategy (reference default on pure meshes, "auto").
//
// _build_offset_blocks (_kernels.py:490-594): on a uniform pure-kind grid
// the pair geometry depends only on the cell offset d and the proto pair,
// so Algorithm 1 runs once per (d, t2, t1) on the reference's synthetic
// geometry (outer cell at the origin, inner cell at d*h) -- one thread per
// block here.  _scatter_offset_blocks (_kernels.py:597-647): every realised
// (inner cell, offset) adds the block; A22 blocks are summed per inner
// element and added once.  Scatter = one warp per inner element of a
// colour, lanes over block entries (race-free, deterministic).
namespace {

struct BlockArgs {
  int kind, nproto, R, nloc;
  double h;
  const double *protos;  // (nproto, 3, 2) triangle protos in cell units
  double *B21, *B22;
  unsigned long long *bev;
  int64_t nblk;
};

template <int DIM, int NLM>
__global__ void __launch_bounds__(128) k_blocks(AsmParams P, BlockArgs B) {
  const MfRules &Rr = P.rules;
  const int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= B.nblk) return;
  const int span = 2 * B.R + 1, np = B.nproto;
  int64_t t = bi;
  const int t1 = (int)(t % np);
  t /= np;
  const int t2 = (int)(t % np);
  t /= np;
  const int ix = (int)(t % span);
  t /= span;
  const int iy = (int)(t % span);
  t /= span;
  const int iz = (int)t;
  const int dx = ix - B.R, dy = iy - B.R, dz = DIM == 3 ? iz - B.R : 0;
  const double h = B.h;
  const double dd[3] = {(double)dx * h, (double)dy * h, (double)dz * h};
  Outer O;
  Inner I;
  I.kind = B.kind == 1 ? 1 : 0;
  O.kind = B.kind;
  O.nloc = I.nloc = B.nloc;
  I.nq = B.kind == 1 ? Rr.nq_tri_in : Rr.nq_box_in;
  I.pts = B.kind == 1 ? Rr.tri_in_pts : Rr.box_in_pts;
  I.w = B.kind == 1 ? Rr.tri_in_w : Rr.box_in_w;
  I.phi = B.kind == 1 ? Rr.phi_tri_in : Rr.phi_box_in;
#pragma unroll
  for (int k = 0; k < DIM; k++) {
    I.lo[k] = dd[k];
    I.hi[k] = xadd(dd[k], h);
  }
  if (B.kind == 1) {
    const double *po = B.protos + t2 * 6, *pi = B.protos + t1 * 6;
    double oc[6], ic[6];
    for (int v = 0; v < 3; v++) {
      oc[2 * v] = xmul(po[2 * v], h);
      oc[2 * v + 1] = xmul(po[2 * v + 1], h);
      ic[2 * v] = xadd(xmul(pi[2 * v], h), dd[0]);
      ic[2 * v + 1] = xadd(xmul(pi[2 * v + 1], h), dd[1]);
    }
    for (int u = 0; u < 6; u++) O.geo[u] = oc[u];
    const double e10 = oc[2] - oc[0], e11 = oc[3] - oc[1];
    const double e20 = oc[4] - oc[0], e21 = oc[5] - oc[1];
    const double det = e10 * e21 - e11 * e20;
    O.v0[0] = oc[0];
    O.v0[1] = oc[1];
    O.inv[0] = e21 / det;
    O.inv[1] = -e20 / det;
    O.inv[2] = -e11 / det;
    O.inv[3] = e10 / det;
    I.c0[0] = ic[0];
    I.c0[1] = ic[1];
    I.e1[0] = xsub(ic[2], ic[0]);
    I.e1[1] = xsub(ic[3], ic[1]);
    I.e2[0] = xsub(ic[4], ic[0]);
    I.e2[1] = xsub(ic[5], ic[1]);
    I.scale_w = I.e1[0] * I.e2[1] - I.e1[1] * I.e2[0];
  } else {
    double jac = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      O.lo[k] = 0.0;
      O.hi[k] = h;
      O.geo[k] = 0.0;
      O.geo[DIM + k] = h;
      jac *= 0.5 * (I.hi[k] - I.lo[k]);
    }
    I.scale_w = jac;
  }
  double mvec[NLM];
  for (int i = 0; i < I.nloc; i++) {
    double s = 0.0;
    for (int q = 0; q < I.nq; q++) s += I.w[q] * I.phi[q * I.nloc + i];
    mvec[i] = s * I.scale_w;
  }
  double *G = P.scratch + bi * P.scratch_stride;
  for (int q = 0; q < I.nq; q++) G[q] = 0.0;
  double Gall = 0.0;
  double b21[NLM * NLM];
  for (int i = 0; i < I.nloc * NLM; i++) b21[i] = 0.0;
  EvCounts cnt = {0, 0, 0, 0};
  const unsigned long long ev =
      pair_run<DIM, NLM>(P, O, I, mvec, b21, G, Gall, cnt);
  const int nl = B.nloc;
  double *o21 = B.B21 + bi * nl * nl, *o22 = B.B22 + bi * nl * nl;
  for (int i = 0; i < nl; i++)
    for (int j = 0; j < nl; j++) {
      o21[i * nl + j] = b21[i * NLM + j];
      o22[i * nl + j] = 0.0;
    }
  if (ev) {
    for (int q = 0; q < I.nq; q++) {
      const double s = (G[q] + Gall) * I.w[q] * I.scale_w;
      if (s == 0.0) continue;
      for (int i = 0; i < nl; i++) {
        const double ci = s * I.phi[q * nl + i];
        for (int j = 0; j < nl; j++) o22[i * nl + j] += ci * I.phi[q * nl + j];
      }
    }
  }
  B.bev[bi] = ev;
}

struct ScatterArgs {
  int nproto, R, nloc, dim;
  const int32_t *blk;  // nonzero block ids sorted by inner proto
  int64_t ptr[3];      // ranges of blk per inner proto (nproto <= 2)
  const double *B21, *B22;
  const unsigned long long *bev;
};

template <int MAXE>
__global__ void __launch_bounds__(128) k_blocked_scatter(AsmParams P,
                                                         ScatterArgs S) {
  const MfMesh &M = P.mesh;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= P.n_inner) return;
  const int64_t m = P.inner[w];
  const int np = S.nproto, nl = S.nloc, ne = nl * nl;
  const int t1 = (int)(m % np);
  const int cell = (int)(m / np);
  int cx, cy, cz;
  cell_coords(cell, M.ncx, M.ncy, cx, cy, cz);
  const int span = 2 * S.R + 1;
  const int64_t *din = M.elem_dofs + m * M.nloc_max;
  double a22[MAXE];
#pragma unroll
  for (int k = 0; k < MAXE; k++) a22[k] = 0.0;
  unsigned long long ev = 0, pairs = 0;
  for (int64_t k = S.ptr[t1]; k < S.ptr[t1 + 1]; k++) {
    const int bi = S.blk[k];
    int t = bi / np;
    const int t2 = t % np;
    t /= np;
    const int dx = t % span - S.R;
    t /= span;
    const int dy = t % span - S.R;
    t /= span;
    const int dz = S.dim == 3 ? t - S.R : 0;
    const int ox = cx - dx, oy = cy - dy, oz = cz - dz;
    if (ox < 0 || ox >= M.ncx || oy < 0 || oy >= M.ncy || oz < 0 ||
        oz >= M.ncz)
      continue;
    const int64_t eo = ((int64_t)(oz * M.ncy + oy) * M.ncx + ox) * np + t2;
    if (!P.outer_mask[eo]) continue;
    ev += S.bev[bi];
    pairs++;
    const int64_t *dout = M.elem_dofs + eo * M.nloc_max;
    const double *b21 = S.B21 + (int64_t)bi * ne;
    const double *b22 = S.B22 + (int64_t)bi * ne;
#pragma unroll
    for (int u = 0; u < MAXE; u++) {
      const int e = lane + 32 * u;
      if (e < ne) {
        const int i = e / nl, j = e - (e / nl) * nl;
        P.vals[pat_index(P.pat, din[i], dout[j])] += P.scale * b21[e];
        a22[u] += b22[e];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < MAXE; u++) {
    const int e = lane + 32 * u;
    if (e < ne && pairs) {
      const int i = e / nl, j = e - (e / nl) * nl;
      P.vals[pat_index(P.pat, din[i], din[j])] += P.scale * a22[u];
    }
  }
  if (lane == 0) {
    counter_add(P.counters + MF_CNT_EVENTS, ev);
    counter_add(P.counters + MF_CNT_PAIRS, pairs);
  }
}

}  // namespace

cudaError_t mf_launch_blocks(const AsmParams &P, int kind, int nproto, int R,
                             double h, const double *protos, double *B21,
                             double *B22, unsigned long long *bev,
                             int64_t nblk, cudaStream_t s) {
  BlockArgs B;
  B.kind = kind;
  B.nproto = nproto;
  B.R = R;
  B.h = h;
  B.protos = protos;
  B.B21 = B21;
  B.B22 = B22;
  B.bev = bev;
  B.nblk = nblk;
  const int dim = P.mesh.dim;
  B.nloc = kind == 1 ? 3 * P.mesh.degree : (dim == 3 ? P.nl_box : P.nl_box);
  const int grid = (int)((nblk + 127) / 128);
  if (dim == 2)
    k_blocks<2, 9><<<grid, 128, 0, s>>>(P, B);
  else if (B.nloc <= 8)
    k_blocks<3, 8><<<grid, 128, 0, s>>>(P, B);
  else
    k_blocks<3, 27><<<grid, 128, 0, s>>>(P, B);
  return cudaGetLastError();
}

cudaError_t mf_launch_blocked_scatter(const AsmParams &P, int nproto, int R,
                                      int nloc, const int32_t *blk,
                                      const int64_t *ptr, const double *B21,
                                      const double *B22,
                                      const unsigned long long *bev,
                                      cudaStream_t s) {
  ScatterArgs S;
  S.nproto = nproto;
  S.R = R;
  S.nloc = nloc;
  S.dim = P.mesh.dim;
  S.blk = blk;
  for (int i = 0; i <= nproto; i++) S.ptr[i] = ptr[i];
  S.B21 = B21;
  S.B22 = B22;
  S.bev = bev;
  const int64_t threads = P.n_inner * 32;
  const int grid = (int)((threads + 127) / 128);
  const int ne = nloc * nloc;
  if (ne <= 32)
    k_blocked_scatter<1><<<grid, 128, 0, s>>>(P, S);
  else if (ne <= 64)
    k_blocked_scatter<2><<<grid, 128, 0, s>>>(P, S);
  else if (ne <= 96)
    k_blocked_scatter<3><<<grid, 128, 0, s>>>(P, S);
  else
    k_blocked_scatter<23><<<grid, 128, 0, s>>>(P, S);
  return cudaGetLastError();
}

// ===========================================================================
// Blocked strategy, gather form (degree 1, pure quad / tri / hex).
//
// vals(r, c) = sum over inner m containing r, outer l containing c of the
// block of offset d = cell(m) - cell(l) (the reference's convention: outer
// cell at the origin, inner at d*h, _kernels.py:531-548, 622-634), entry
// (i(r in m), j(c in l)), plus A22acc[m][i][j(c in m)] when c is a DOF of
// m -- exactly the sum _scatter_offset_blocks accumulates
// (_kernels.py:597-647), evaluated entry by entry.  Each value is written
// once (coalesced, deterministic, no read-modify-write, no colouring).
//
// Elements holding a DOF are enumerated as "combos" u = (cell offset a_u,
// proto t_u, local index i_u): 8 for hexes, 4 for quads, 6 for triangles.
// With r's combo u and c's combo v, d = b_v - a_u - (c - r), so for a fixed
// (u, v) the lanes of a warp (consecutive columns of one row) read
// consecutive words of T[u][v][d] -- the block entries re-laid out with
// the offset innermost and zero-padded to |d| <= R+2 (absent blocks are
// exactly zero).  A22acc of elements whose whole offset box is realised is
// one constant per proto, computed once.
namespace {

#ifndef MF_BLOCKED_STENCIL
#define MF_BLOCKED_STENCIL 1
#endif

struct Combo {
  int ax, ay, az, t, i;
};

// combos of a DOF (degree 1): element (cell = dof - a, proto t) carries it
// as local index i (fe_space.py:68-80)
MF_DEV int dof_combos(int kind, int dim, Combo *cb) {
  int n = 0;
  if (kind == 1) {  // lower (0,0)(1,0)(1,1), upper (0,0)(1,1)(0,1)
    const int tab[6][4] = {{0, 0, 0, 0}, {1, 0, 0, 1}, {1, 1, 0, 2},
                           {0, 0, 1, 0}, {1, 1, 1, 1}, {0, 1, 1, 2}};
    for (int k = 0; k < 6; k++)
      cb[n++] = {tab[k][0], tab[k][1], 0, tab[k][2], tab[k][3]};
    return n;
  }
  const int az = dim == 3 ? 1 : 0;
  for (int z = 0; z <= az; z++)
    for (int y = 0; y <= 1; y++)
      for (int x = 0; x <= 1; x++) cb[n++] = {x, y, z, 0, x + 2 * y + 4 * z};
  return n;
}

MF_DEV int64_t block_id(int R, int np, int dim, int dx, int dy, int dz,
                        int t2, int t1) {
  const int span = 2 * R + 1;
  const int iz = dim == 3 ? dz + R : 0;
  return ((((int64_t)iz * span + (dy + R)) * span + (dx + R)) * np + t2) *
             np + t1;
}

struct GatherArgs {
  int nproto, R, nloc, dim, kind, ncombo, P2;  // P2 = 2R+5 (padded span)
  int64_t row0, row1;
  // interior rows (every element holding r or any of its columns exists,
  // row box unclipped) are translates of one another: their values are
  // one stencil, gathered once for a reference row and copied
  const double *stencil;   // NULL: gather every row
  int in_lo[3], in_hi[3];  // interior DOF box per axis (inclusive)
  double *row_out;         // non-NULL: write the (single) row here
  const double *B21, *B22;
  const unsigned long long *bev;
  double *T;          // (ncombo, ncombo, P2^dim)
  double *a22;        // (n_elem, nloc, nloc)
  double *a22full;    // (nproto, nloc, nloc)
};

// T[u][v][d] = B21[block(d, t_v, t_u)][i_u][j_v], zero outside |d| <= R
__global__ void k_build_T(GatherArgs G) {
  const int64_t vol = G.dim == 3 ? (int64_t)G.P2 * G.P2 * G.P2
                                 : (int64_t)G.P2 * G.P2;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)G.ncombo * G.ncombo * vol) return;
  Combo cb[8];
  dof_combos(G.kind, G.dim, cb);
  const int u = (int)(k / (G.ncombo * vol));
  const int v = (int)((k / vol) % G.ncombo);
  int64_t rem = k % vol;
  const int h = G.R + 2;
  const int dx = (int)(rem % G.P2) - h;
  rem /= G.P2;
  const int dy = (int)(rem % G.P2) - h;
  const int dz = G.dim == 3 ? (int)(rem / G.P2) - h : 0;
  double val = 0.0;
  if (abs(dx) <= G.R && abs(dy) <= G.R && abs(dz) <= G.R) {
    const int64_t b = block_id(G.R, G.nproto, G.dim, dx, dy, dz, cb[v].t,
                               cb[u].t);
    if (G.bev[b])
      val = G.B21[b * G.nloc * G.nloc + cb[u].i * G.nloc + cb[v].i];
  }
  G.T[k] = val;
}

// A22acc of a fully realised element, per proto (one warp)
__global__ void k_a22_full(GatherArgs G) {
  const int lane = threadIdx.x;
  const int np = G.nproto, ne = G.nloc * G.nloc;
  const int zr = G.dim == 3 ? G.R : 0;
  for (int t1 = 0; t1 < np; t1++)
    for (int e = lane; e < ne; e += 32) {
      double acc = 0.0;
      for (int dz = -zr; dz <= zr; dz++)
        for (int dy = -G.R; dy <= G.R; dy++)
          for (int dx = -G.R; dx <= G.R; dx++)
            for (int t2 = 0; t2 < np; t2++) {
              const int64_t b = block_id(G.R, np, G.dim, dx, dy, dz, t2, t1);
              if (G.bev[b]) acc += G.B22[b * ne + e];
            }
      G.a22full[t1 * ne + e] = acc;
    }
}

// per element: A22acc (boundary elements loop over their realised offset
// box, interior ones copy the constant) and the realised events / pairs
__global__ void __launch_bounds__(128) k_blocked_a22(AsmParams P,
                                                     GatherArgs G) {
  const MfMesh &M = P.mesh;
  const int lane = threadIdx.x & 31;
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (m >= M.n_elem) return;
  const int np = G.nproto, ne = G.nloc * G.nloc;
  const int t1 = (int)(m % np);
  int cx, cy, cz;
  cell_coords((int)(m / np), M.ncx, M.ncy, cx, cy, cz);
  const int zr = G.dim == 3 ? G.R : 0;
  // realised offsets: outer cell (c - d) inside the grid
  const int dxlo = max(-G.R, cx - (M.ncx - 1)), dxhi = min(G.R, cx);
  const int dylo = max(-G.R, cy - (M.ncy - 1)), dyhi = min(G.R, cy);
  const int dzlo = max(-zr, cz - (M.ncz - 1)), dzhi = min(zr, cz);
  const bool full = dxlo == -G.R && dxhi == G.R && dylo == -G.R &&
                    dyhi == G.R && dzlo == -zr && dzhi == zr;
  double acc[2] = {0.0, 0.0};
  unsigned long long ev = 0, pairs = 0;
  for (int dz = dzlo; dz <= dzhi; dz++)
    for (int dy = dylo; dy <= dyhi; dy++)
      for (int dx = dxlo; dx <= dxhi; dx++)
        for (int t2 = 0; t2 < np; t2++) {
          const int64_t b = block_id(G.R, np, G.dim, dx, dy, dz, t2, t1);
          const unsigned long long e = G.bev[b];
          if (!e) continue;
          ev += e;
          pairs++;
          if (!full) {
            const double *b22 = G.B22 + b * ne;
            for (int u = 0; u < 2; u++) {
              const int k = lane + 32 * u;
              if (k < ne) acc[u] += b22[k];
            }
          }
        }
  double *out = G.a22 + m * ne;
  for (int u = 0; u < 2; u++) {
    const int k = lane + 32 * u;
    if (k < ne) out[k] = full ? G.a22full[t1 * ne + k] : acc[u];
  }
  if (lane == 0) {
    counter_add(P.counters + MF_CNT_EVENTS, ev);
    counter_add(P.counters + MF_CNT_PAIRS, pairs);
  }
}

// one warp per DOF row, lanes over the row's entries
__global__ void __launch_bounds__(256) k_blocked_gather(AsmParams P,
                                                        GatherArgs G) {
  const MfMesh &M = P.mesh;
  const MfPattern &Pt = P.pat;
  const int lane = threadIdx.x & 31;
  const int64_t r =
      G.row0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (r >= G.row1) return;
  const int np = G.nproto, nl = G.nloc, ne = nl * nl, nc = G.ncombo;
  const int rx = (int)(r % Pt.NX);
  const int64_t rt = r / Pt.NX;
  const int ry = (int)(rt % Pt.NY), rz = (int)(rt / Pt.NY);
  const int xlo = max(rx - Pt.K, 0), xhi = min(rx + Pt.K, Pt.NX - 1);
  const int ylo = max(ry - Pt.K, 0), yhi = min(ry + Pt.K, Pt.NY - 1);
  const int zlo = max(rz - Pt.K, 0), zhi = min(rz + Pt.K, Pt.NZ - 1);
  const int Wx = xhi - xlo + 1, Wy = yhi - ylo + 1;
  const int nent = Wx * Wy * (zhi - zlo + 1);
  const int64_t p0 = Pt.rowptr[r];
  if (G.stencil && rx >= G.in_lo[0] && rx <= G.in_hi[0] &&
      ry >= G.in_lo[1] && ry <= G.in_hi[1] && rz >= G.in_lo[2] &&
      rz <= G.in_hi[2]) {
    // the same block lookups in the same order as the reference row:
    // bit-identical values, written at HBM speed
    for (int k = lane; k < nent; k += 32) P.vals[p0 + k] = G.stencil[k];
    return;
  }
  Combo cb[8];
  dof_combos(G.kind, G.dim, cb);
  // inner elements holding r (uniform per warp)
  unsigned mexist = 0;
  int64_t melem[8];
#pragma unroll
  for (int u = 0; u < 8; u++) {
    melem[u] = 0;
    if (u < nc) {
      const int ccx = rx - cb[u].ax, ccy = ry - cb[u].ay, ccz = rz - cb[u].az;
      if (ccx >= 0 && ccx < M.ncx && ccy >= 0 && ccy < M.ncy && ccz >= 0 &&
          ccz < M.ncz) {
        mexist |= 1u << u;
        melem[u] = ((int64_t)(ccz * M.ncy + ccy) * M.ncx + ccx) * np +
                   cb[u].t;
      }
    }
  }
  const int h = G.R + 2, P2 = G.P2;
  const int64_t vol = G.dim == 3 ? (int64_t)P2 * P2 * P2 : (int64_t)P2 * P2;
  for (int k = lane; k < nent; k += 32) {
    const int ix = k % Wx;
    const int tt = k / Wx;
    const int cxg = xlo + ix, cyg = ylo + tt % Wy, czg = zlo + tt / Wy;
    const int Dx = cxg - rx, Dy = cyg - ry, Dz = czg - rz;
    // outer elements holding c
    unsigned lexist = 0;
#pragma unroll
    for (int v = 0; v < 8; v++) {
      if (v < nc) {
        const int lx = cxg - cb[v].ax, ly = cyg - cb[v].ay,
                  lz = czg - cb[v].az;
        if (lx >= 0 && lx < M.ncx && ly >= 0 && ly < M.ncy && lz >= 0 &&
            lz < M.ncz)
          lexist |= 1u << v;
      }
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (u >= nc || !((mexist >> u) & 1u)) continue;
      const double *Tu = G.T + (int64_t)u * nc * vol;
#pragma unroll
      for (int v = 0; v < 8; v++) {
        if (v >= nc || !((lexist >> v) & 1u)) continue;
        const int dx = cb[v].ax - cb[u].ax - Dx + h;
        const int dy = cb[v].ay - cb[u].ay - Dy + h;
        const int dz = G.dim == 3 ? cb[v].az - cb[u].az - Dz + h : 0;
        s += Tu[v * vol + ((int64_t)dz * P2 + dy) * P2 + dx];
      }
      // A22: c a DOF of m itself
      const int ox = Dx + cb[u].ax, oy = Dy + cb[u].ay, oz = Dz + cb[u].az;
      if (ox >= 0 && ox <= 1 && oy >= 0 && oy <= 1 && oz >= 0 &&
          oz <= (G.dim == 3 ? 1 : 0)) {
        int j = -1;
        for (int w = 0; w < nc; w++)
          if (cb[w].t == cb[u].t && cb[w].ax == ox && cb[w].ay == oy &&
              cb[w].az == oz)
            j = cb[w].i;
        if (j >= 0) s += G.a22[melem[u] * ne + cb[u].i * nl + j];
      }
    }
    if (G.row_out)
      G.row_out[k] = P.scale * s;
    else
      P.vals[p0 + k] = P.scale * s;
  }
}

GatherArgs gather_args(const AsmParams &P, int kind, int nproto, int R,
                       const double *B21, const double *B22,
                       const unsigned long long *bev, double *T, double *a22,
                       double *a22full) {
  GatherArgs G;
  G.nproto = nproto;
  G.R = R;
  G.dim = P.mesh.dim;
  G.kind = kind;
  G.nloc = kind == 1 ? 3 : (P.mesh.dim == 3 ? 8 : 4);
  G.ncombo = kind == 1 ? 6 : (P.mesh.dim == 3 ? 8 : 4);
  G.P2 = 2 * R + 5;
  G.B21 = B21;
  G.B22 = B22;
  G.bev = bev;
  G.T = T;
  G.a22 = a22;
  G.a22full = a22full;
  G.row0 = 0;
  G.row1 = P.pat.n;
  G.stencil = nullptr;
  G.row_out = nullptr;
  for (int k = 0; k < 3; k++) {
    G.in_lo[k] = 0;
    G.in_hi[k] = -1;
  }
  return G;
}

}  // namespace

// workspace doubles: T + a22full (a22 is separate)
int64_t mf_gather_table_doubles(int dim, int kind, int R) {
  const int64_t P2 = 2 * R + 5;
  const int nc = kind == 1 ? 6 : (dim == 3 ? 8 : 4);
  const int nl = kind == 1 ? 3 : (dim == 3 ? 8 : 4);
  return (int64_t)nc * nc * (dim == 3 ? P2 * P2 * P2 : P2 * P2) +
         2 * nl * nl;
}

cudaError_t mf_launch_blocked_a22(const AsmParams &P, int kind, int nproto,
                                  int R, const double *B21, const double *B22,
                                  const unsigned long long *bev, double *a22,
                                  double *table, cudaStream_t s) {
  const int64_t tsz = mf_gather_table_doubles(P.mesh.dim, kind, R);
  const int nl = kind == 1 ? 3 : (P.mesh.dim == 3 ? 8 : 4);
  GatherArgs G = gather_args(P, kind, nproto, R, B21, B22, bev, table, a22,
                             table + tsz - 2 * nl * nl);
  const int64_t nT = tsz - 2 * nl * nl;
  k_build_T<<<(unsigned)((nT + 255) / 256), 256, 0, s>>>(G);
  k_a22_full<<<1, 32, 0, s>>>(G);
  const int64_t t = P.mesh.n_elem * 32;
  if (t > 0)
    k_blocked_a22<<<(unsigned)((t + 127) / 128), 128, 0, s>>>(P, G);
  return cudaGetLastError();
}

cudaError_t mf_launch_blocked_gather(const AsmParams &P, int kind, int nproto,
                                     int R, const double *table,
                                     const double *a22, int64_t row0,
                                     int64_t row1, cudaStream_t s) {
  GatherArgs G = gather_args(P, kind, nproto, R, nullptr, nullptr, nullptr,
                             const_cast<double *>(table),
                             const_cast<double *>(a22), nullptr);
  G.row0 = row0;
  G.row1 = row1;
  const int64_t t = (row1 - row0) * 32;
  if (t <= 0) return cudaGetLastError();
  // interior DOF box: r - K - 1 >= 0 and r + K <= N - 2 on every axis
  // (elements around r and around every column c exist; row box unclipped)
  const MfPattern &Pt = P.pat;
  const int K = Pt.K, N[3] = {Pt.NX, Pt.NY, Pt.NZ};
  bool interior = MF_BLOCKED_STENCIL != 0;
  for (int k = 0; k < 3; k++) {
    if (k == 2 && P.mesh.dim == 2) {
      G.in_lo[2] = 0;
      G.in_hi[2] = 0;
      continue;
    }
    G.in_lo[k] = K + 1;
    G.in_hi[k] = N[k] - 2 - K;
    if (G.in_lo[k] > G.in_hi[k]) interior = false;
  }
  double *stencil = nullptr;
  if (interior) {
    const int span = 2 * K + 1;
    const int64_t nent = (int64_t)span * span * (P.mesh.dim == 3 ? span : 1);
    cudaError_t e = cudaMallocAsync(&stencil, sizeof(double) * nent, s);
    if (e != cudaSuccess) return e;
    // reference row: the centre of the interior box, gathered into the
    // scratch
    const int cx = (G.in_lo[0] + G.in_hi[0]) / 2;
    const int cy = (G.in_lo[1] + G.in_hi[1]) / 2;
    const int cz = (G.in_lo[2] + G.in_hi[2]) / 2;
    const int64_t r0 = ((int64_t)cz * Pt.NY + cy) * Pt.NX + cx;
    GatherArgs G0 = G;
    G0.row0 = r0;
    G0.row1 = r0 + 1;
    G0.row_out = stencil;
    k_blocked_gather<<<1, 32, 0, s>>>(P, G0);
    G.stencil = stencil;
  }
  k_blocked_gather<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(P, G);
  cudaError_t e = cudaGetLastError();
  if (stencil) {
    cudaError_t ef = cudaFreeAsync(stencil, s);
    if (e == cudaSuccess) e = ef;
  }
  return e;
}
