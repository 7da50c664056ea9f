/*
 * mf_oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg are the only callers.  The product
 * path (paper_2101_08825_b200) never links or loads this library.
 *
 * Restates the numba cores of the reference package mollifem
 * (/root/reference/pkg/src/mollifem/_kernels.py) in plain C, statement by
 * statement and in the same floating-point evaluation order, so that with
 * -ffp-contract=off (no FMA; the numba build has none either, SURVEY.md
 * section 0 fact 4) the results are bit-identical to the reference:
 *
 *   mu2                 _kernels.py:18-29
 *   shape1d / shape_at  _kernels.py:32-77
 *   aprx_min / max      _kernels.py:80-102
 *   event_box           _kernels.py:105-143
 *   event_tri           _kernels.py:146-181
 *   pair_blocks         _kernels.py:184-313  (Algorithm 1, LIFO stack)
 *   inner_data          _kernels.py:316-340
 *   tri_inv             _kernels.py:343-355
 *   scatter_block       _kernels.py:358-388
 *   general_core        _kernels.py:391-487
 *   eidx / matvec / symmetrize / asymmetry_inf / diag
 *                       _kernels.py:846-957, 1199-1202
 *   count / fill candidates  _kernels.py:1205-1268
 *
 * Pinned against the live reference by tests/golden (bit-exact vals,
 * events and candidate lists; see tests/golden/make_golden.py).
 *
 * Tetrahedra (element kind 3, P1) are NEW: the
 * reference has no tet element, so event_tet / tet_inv / the 8-child split
 * below extend Algorithm 1 in the reference's style (box distances on the
 * sub-cell's vertex bounding box, rank-1 event form, midpoint children by
 * Bey's red refinement).  Parity for tets is unpinned against the
 * reference; tests/test_tet.py pins it by identities instead (A 1 = 0,
 * symmetry, quadrature convergence) and checks the GPU against this code.
 * In 3D the "tri" rule slots carry the tet rule (points nq x 3).
 *
 * Extra over the reference (instrumentation only, does not change any
 * arithmetic): an optional event census and a pthread driver that runs
 * disjoint outer-element subsets concurrently (the reference's
 * parallel_assemble thread pool over nogil numba, parallel.py:174-178) for
 * the CPU baseline timing.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define STACK_CAP 256

static inline double pymin(double a, double b) { return (b < a) ? b : a; }
static inline double pymax(double a, double b) { return (b > a) ? b : a; }

static inline double mu2(double d2, double dm2, double dp2, double delta,
                         double eps) {
  if (d2 <= dm2) return 1.0;
  if (d2 >= dp2) return 0.0;
  double r = (delta - sqrt(d2)) / eps;
  double r2 = r * r;
  return (((((35.0 * r2 - 180.0) * r2 + 378.0) * r2 - 420.0) * r2 + 315.0) *
              r + 128.0) / 256.0;
}

static inline void shape1d(int degree, double t, double *out) {
  if (degree == 1) {
    out[0] = 0.5 * (1.0 - t);
    out[1] = 0.5 * (1.0 + t);
  } else {
    out[0] = 0.5 * t * (t - 1.0);
    out[1] = 1.0 - t * t;
    out[2] = 0.5 * t * (t + 1.0);
  }
}

/* kind: 0 quad, 1 tri, 2 hex, 3 tet (P1 only) */
static int shape_at(int kind, int degree, int dim, double r0, double r1,
                    double r2, double *out) {
  if (kind == 3) {
    out[0] = ((1.0 - r0) - r1) - r2;
    out[1] = r0; out[2] = r1; out[3] = r2;
    return 4;
  }
  if (kind == 1) {
    double la = 1.0 - r0 - r1;
    if (degree == 1) {
      out[0] = la; out[1] = r0; out[2] = r1;
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

static inline double aprx_min(const double *alo, const double *ahi,
                              const double *blo, const double *bhi, int dim) {
  double m = 0.0;
  for (int k = 0; k < dim; k++) {
    double d1 = alo[k] - bhi[k];
    double d2 = blo[k] - ahi[k];
    if (d1 > m) m = d1;
    if (d2 > m) m = d2;
  }
  return m;
}

static inline double aprx_max(const double *alo, const double *ahi,
                              const double *blo, const double *bhi, int dim) {
  double s = 0.0;
  for (int k = 0; k < dim; k++) {
    double d1 = alo[k] - bhi[k];
    double d2 = blo[k] - ahi[k];
    double a = d1 * d1, b = d2 * d2;
    s += (a > b) ? a : b;
  }
  return sqrt(s);
}

/* census helper: exact Euclidean gap between boxes (instrumentation) */
static inline double box_gap_euclid(const double *alo, const double *ahi,
                                    const double *blo, const double *bhi,
                                    int dim) {
  double s = 0.0;
  for (int k = 0; k < dim; k++) {
    double g = alo[k] - bhi[k];
    double g2 = blo[k] - ahi[k];
    if (g2 > g) g = g2;
    if (g < 0.0) g = 0.0;
    s += g * g;
  }
  return sqrt(s);
}

typedef struct {
  int dim, degree;
  const double *box_pts, *box_w;  /* outer box rule */
  int nq_box;
  const double *tri_pts, *tri_w;  /* outer tri rule */
  int nq_tri;
  double delta, eps, cde, dm2, dp2, dme, dpe;
  int L_min, L_max;
  int64_t *census;
} Ctx;

static void event_box(const Ctx *c, int okind, const double *g,
                      const double *o_lo, const double *o_hi,
                      const double *y1, const double *w1, int nq1,
                      const double *PHI1, int nloc1, double *b21, int ldb,
                      double *gsum, int nloc2) {
  int dim = c->dim;
  double phi2[27];
  double jac = 1.0;
  for (int k = 0; k < dim; k++) jac *= 0.5 * (g[dim + k] - g[k]);
  for (int q2 = 0; q2 < c->nq_box; q2++) {
    const double *pt = c->box_pts + (size_t)q2 * dim;
    double x0 = g[0] + (pt[0] + 1.0) * 0.5 * (g[dim] - g[0]);
    double x1 = g[1] + (pt[1] + 1.0) * 0.5 * (g[dim + 1] - g[1]);
    double x2 = 0.0;
    if (dim == 3) x2 = g[2] + (pt[2] + 1.0) * 0.5 * (g[5] - g[2]);
    double w2q = c->box_w[q2] * jac;
    double rx = (x0 - o_lo[0]) / (o_hi[0] - o_lo[0]) * 2.0 - 1.0;
    double ry = (x1 - o_lo[1]) / (o_hi[1] - o_lo[1]) * 2.0 - 1.0;
    double rz = 0.0;
    if (dim == 3) rz = (x2 - o_lo[2]) / (o_hi[2] - o_lo[2]) * 2.0 - 1.0;
    shape_at(okind, c->degree, dim, rx, ry, rz, phi2);
    for (int q1 = 0; q1 < nq1; q1++) {
      double dx = x0 - y1[q1 * 3 + 0];
      double dy = x1 - y1[q1 * 3 + 1];
      double d2 = dx * dx + dy * dy;
      if (dim == 3) {
        double dz = x2 - y1[q1 * 3 + 2];
        d2 += dz * dz;
      }
      if (d2 >= c->dp2) {
        if (c->census) c->census[6]++;
        continue;
      }
      if (c->census) c->census[d2 <= c->dm2 ? 4 : 5]++;
      double gam = c->cde * mu2(d2, c->dm2, c->dp2, c->delta, c->eps);
      double tq = gam * w2q;
      gsum[q1] += tq;
      double tw = tq * w1[q1];
      for (int i = 0; i < nloc1; i++) {
        double ci = tw * PHI1[q1 * nloc1 + i];
        for (int j = 0; j < nloc2; j++) b21[i * ldb + j] -= ci * phi2[j];
      }
    }
  }
}

static void event_tri(const Ctx *c, const double *g, const double *o_v0,
                      const double *o_inv, const double *y1,
                      const double *w1, int nq1, const double *PHI1,
                      int nloc1, double *b21, int ldb, double *gsum,
                      int nloc2) {
  double phi2[27];
  double e10 = g[2] - g[0];
  double e11 = g[3] - g[1];
  double e20 = g[4] - g[0];
  double e21 = g[5] - g[1];
  double det = e10 * e21 - e11 * e20;
  for (int q2 = 0; q2 < c->nq_tri; q2++) {
    double px = c->tri_pts[q2 * 2 + 0];
    double py = c->tri_pts[q2 * 2 + 1];
    double x0 = g[0] + px * e10 + py * e20;
    double x1 = g[1] + px * e11 + py * e21;
    double w2q = c->tri_w[q2] * det;
    double dx0 = x0 - o_v0[0];
    double dx1 = x1 - o_v0[1];
    double rx = o_inv[0] * dx0 + o_inv[1] * dx1;
    double ry = o_inv[2] * dx0 + o_inv[3] * dx1;
    shape_at(1, c->degree, 2, rx, ry, 0.0, phi2);
    for (int q1 = 0; q1 < nq1; q1++) {
      double dx = x0 - y1[q1 * 3 + 0];
      double dy = x1 - y1[q1 * 3 + 1];
      double d2 = dx * dx + dy * dy;
      if (d2 >= c->dp2) {
        if (c->census) c->census[6]++;
        continue;
      }
      if (c->census) c->census[d2 <= c->dm2 ? 4 : 5]++;
      double gam = c->cde * mu2(d2, c->dm2, c->dp2, c->delta, c->eps);
      double tq = gam * w2q;
      gsum[q1] += tq;
      double tw = tq * w1[q1];
      for (int i = 0; i < nloc1; i++) {
        double ci = tw * PHI1[q1 * nloc1 + i];
        for (int j = 0; j < nloc2; j++) b21[i * ldb + j] -= ci * phi2[j];
      }
    }
  }
}

/* tet edge vectors from vertex 0 of g (12 doubles) and the determinant
 * e1 . (e2 x e3) in a fixed order (shared by event_tet, tet_inv and
 * inner_data) */
static inline double tet_edges(const double *g, double *e1, double *e2,
                               double *e3) {
  for (int k = 0; k < 3; k++) {
    e1[k] = g[3 + k] - g[k];
    e2[k] = g[6 + k] - g[k];
    e3[k] = g[9 + k] - g[k];
  }
  double c0 = e2[1] * e3[2] - e2[2] * e3[1];
  double c1 = e2[2] * e3[0] - e2[0] * e3[2];
  double c2 = e2[0] * e3[1] - e2[1] * e3[0];
  return (e1[0] * c0 + e1[1] * c1) + e1[2] * c2;
}

/* event on sub-tet g: outer points mapped affinely, weights times |det|,
 * pulled back through the outer element's inverse map (o_v0, o_inv 3x3) */
static void event_tet(const Ctx *c, const double *g, const double *o_v0,
                      const double *o_inv, const double *y1,
                      const double *w1, int nq1, const double *PHI1,
                      int nloc1, double *b21, int ldb, double *gsum) {
  double phi2[4], e1[3], e2[3], e3[3];
  double det = fabs(tet_edges(g, e1, e2, e3));
  for (int q2 = 0; q2 < c->nq_tri; q2++) {
    const double *pt = c->tri_pts + (size_t)q2 * 3;
    double x[3];
    for (int k = 0; k < 3; k++)
      x[k] = ((g[k] + pt[0] * e1[k]) + pt[1] * e2[k]) + pt[2] * e3[k];
    double w2q = c->tri_w[q2] * det;
    double d0 = x[0] - o_v0[0], d1 = x[1] - o_v0[1], d2v = x[2] - o_v0[2];
    double rx = (o_inv[0] * d0 + o_inv[1] * d1) + o_inv[2] * d2v;
    double ry = (o_inv[3] * d0 + o_inv[4] * d1) + o_inv[5] * d2v;
    double rz = (o_inv[6] * d0 + o_inv[7] * d1) + o_inv[8] * d2v;
    shape_at(3, 1, 3, rx, ry, rz, phi2);
    for (int q1 = 0; q1 < nq1; q1++) {
      double dx = x[0] - y1[q1 * 3 + 0];
      double dy = x[1] - y1[q1 * 3 + 1];
      double dz = x[2] - y1[q1 * 3 + 2];
      double d2 = (dx * dx + dy * dy) + dz * dz;
      if (d2 >= c->dp2) {
        if (c->census) c->census[6]++;
        continue;
      }
      if (c->census) c->census[d2 <= c->dm2 ? 4 : 5]++;
      double gam = c->cde * mu2(d2, c->dm2, c->dp2, c->delta, c->eps);
      double tq = gam * w2q;
      gsum[q1] += tq;
      double tw = tq * w1[q1];
      for (int i = 0; i < nloc1; i++) {
        double ci = tw * PHI1[q1 * nloc1 + i];
        for (int j = 0; j < 4; j++) b21[i * ldb + j] -= ci * phi2[j];
      }
    }
  }
}

/* the 8 children of a tet by red refinement (Bey): 4 corner tets and the
 * interior octahedron cut along the m02-m13 diagonal; vertex lists index
 * P = {x0, x1, x2, x3, m01, m02, m03, m12, m13, m23} */
static const int TET_CHILD[8][4] = {{0, 4, 5, 6}, {4, 1, 7, 8}, {5, 7, 2, 9},
                                    {6, 8, 9, 3}, {4, 5, 6, 8}, {4, 5, 7, 8},
                                    {5, 6, 8, 9}, {5, 7, 8, 9}};

static void tet_children(const double *g, double (*out)[12]) {
  double P[10][3];
  static const int E[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int v = 0; v < 4; v++)
    for (int k = 0; k < 3; k++) P[v][k] = g[3 * v + k];
  for (int e = 0; e < 6; e++)
    for (int k = 0; k < 3; k++)
      P[4 + e][k] = 0.5 * (g[3 * E[e][0] + k] + g[3 * E[e][1] + k]);
  for (int b = 0; b < 8; b++)
    for (int v = 0; v < 4; v++)
      for (int k = 0; k < 3; k++) out[b][3 * v + k] = P[TET_CHILD[b][v]][k];
}

/* Algorithm 1 for one (outer, inner) pair; returns the event count. */
static int64_t pair_blocks(const Ctx *c, int okind, const double *ogeo,
                           const double *o_lo, const double *o_hi,
                           const double *o_v0, const double *o_inv,
                           const double *y1, const double *w1, int nq1,
                           const double *PHI1, int nloc1, const double *i_lo,
                           const double *i_hi, double *b21, double *b22,
                           int ldb, int nloc2, double *gsum,
                           double (*stack_geo)[12], int *stack_lvl) {
  int dim = c->dim;
  int64_t events = 0;
  double slo[3], shi[3], g[12];
  for (int t = 0; t < 12; t++) stack_geo[0][t] = ogeo[t];
  stack_lvl[0] = 1;
  int top = 1;
  for (int q1 = 0; q1 < nq1; q1++) gsum[q1] = 0.0;
  while (top > 0) {
    top -= 1;
    for (int t = 0; t < 12; t++) g[t] = stack_geo[top][t];
    int L = stack_lvl[top];
    if (okind == 3) {
      for (int k = 0; k < 3; k++) {
        slo[k] = pymin(g[k], pymin(g[3 + k], pymin(g[6 + k], g[9 + k])));
        shi[k] = pymax(g[k], pymax(g[3 + k], pymax(g[6 + k], g[9 + k])));
      }
    } else if (okind == 1) {
      slo[0] = pymin(g[0], pymin(g[2], g[4]));
      shi[0] = pymax(g[0], pymax(g[2], g[4]));
      slo[1] = pymin(g[1], pymin(g[3], g[5]));
      shi[1] = pymax(g[1], pymax(g[3], g[5]));
    } else {
      for (int k = 0; k < dim; k++) {
        slo[k] = g[k];
        shi[k] = g[dim + k];
      }
    }
    int do_split = 0, integrate = 0;
    if (L < c->L_min) {
      do_split = 1;
    } else if (L == c->L_max) {
      if (aprx_min(slo, shi, i_lo, i_hi, dim) < c->dpe) integrate = 2;
    } else {
      if (aprx_max(slo, shi, i_lo, i_hi, dim) < c->dme)
        integrate = 1;
      else if (aprx_min(slo, shi, i_lo, i_hi, dim) < c->dpe)
        do_split = 1;
    }
    if (integrate) {
      events += 1;
      if (c->census) {
        if (integrate == 1)
          c->census[0]++;
        else if (aprx_max(slo, shi, i_lo, i_hi, dim) < c->dme)
          c->census[1]++;
        else if (box_gap_euclid(slo, shi, i_lo, i_hi, dim) >= c->dpe)
          c->census[2]++;
        else
          c->census[3]++;
      }
      if (okind == 3)
        event_tet(c, g, o_v0, o_inv, y1, w1, nq1, PHI1, nloc1, b21, ldb,
                  gsum);
      else if (okind == 1)
        event_tri(c, g, o_v0, o_inv, y1, w1, nq1, PHI1, nloc1, b21, ldb,
                  gsum, nloc2);
      else
        event_box(c, okind, g, o_lo, o_hi, y1, w1, nq1, PHI1, nloc1, b21,
                  ldb, gsum, nloc2);
    }
    if (do_split) {
      if (okind == 3) {
        tet_children(g, stack_geo + top);
        for (int b = 0; b < 8; b++) stack_lvl[top + b] = L + 1;
        top += 8;
      } else if (okind == 1) {
        double m010 = 0.5 * (g[0] + g[2]);
        double m011 = 0.5 * (g[1] + g[3]);
        double m120 = 0.5 * (g[2] + g[4]);
        double m121 = 0.5 * (g[3] + g[5]);
        double m200 = 0.5 * (g[4] + g[0]);
        double m201 = 0.5 * (g[5] + g[1]);
        double ch[4][6] = {{g[0], g[1], m010, m011, m200, m201},
                           {m010, m011, g[2], g[3], m120, m121},
                           {m200, m201, m120, m121, g[4], g[5]},
                           {m010, m011, m120, m121, m200, m201}};
        for (int b = 0; b < 4; b++) {
          for (int t = 0; t < 6; t++) stack_geo[top + b][t] = ch[b][t];
          stack_lvl[top + b] = L + 1;
        }
        top += 4;
      } else {
        int nchild = 1 << dim;
        for (int b = 0; b < nchild; b++) {
          for (int k = 0; k < dim; k++) {
            double lo = g[k], hi = g[dim + k];
            double mid = 0.5 * (lo + hi);
            if (((b >> k) & 1) == 0) {
              stack_geo[top + b][k] = lo;
              stack_geo[top + b][dim + k] = mid;
            } else {
              stack_geo[top + b][k] = mid;
              stack_geo[top + b][dim + k] = hi;
            }
          }
          stack_lvl[top + b] = L + 1;
        }
        top += nchild;
      }
    }
  }
  if (events > 0) {
    for (int q1 = 0; q1 < nq1; q1++) {
      double s = gsum[q1] * w1[q1];
      if (s == 0.0) continue;
      for (int i = 0; i < nloc1; i++) {
        double ci = s * PHI1[q1 * nloc1 + i];
        for (int j = 0; j < nloc1; j++)
          b22[i * ldb + j] += ci * PHI1[q1 * nloc1 + j];
      }
    }
  }
  return events;
}

static int inner_data(int dim, int kind, const double *coords, int nv_max,
                      const double *lo, const double *hi,
                      const double *box_pts, const double *box_w, int nq_box,
                      const double *tri_pts, const double *tri_w, int nq_tri,
                      double *y1, double *w1) {
  if (kind == 3) {
    double e1[3], e2[3], e3[3];
    double det = fabs(tet_edges(coords, e1, e2, e3));
    for (int q = 0; q < nq_tri; q++) {
      const double *pt = tri_pts + (size_t)q * 3;
      for (int k = 0; k < 3; k++)
        y1[q * 3 + k] =
            ((coords[k] + pt[0] * e1[k]) + pt[1] * e2[k]) + pt[2] * e3[k];
      w1[q] = tri_w[q] * det;
    }
    return nq_tri;
  }
  if (kind == 1) {
    const double *c0 = coords, *c1 = coords + dim, *c2 = coords + 2 * dim;
    double e10 = c1[0] - c0[0];
    double e11 = c1[1] - c0[1];
    double e20 = c2[0] - c0[0];
    double e21 = c2[1] - c0[1];
    double det = e10 * e21 - e11 * e20;
    for (int q = 0; q < nq_tri; q++) {
      y1[q * 3 + 0] = c0[0] + tri_pts[q * 2] * e10 + tri_pts[q * 2 + 1] * e20;
      y1[q * 3 + 1] = c0[1] + tri_pts[q * 2] * e11 + tri_pts[q * 2 + 1] * e21;
      w1[q] = tri_w[q] * det;
    }
    (void)nv_max;
    return nq_tri;
  }
  double jac = 1.0;
  for (int k = 0; k < dim; k++) jac *= 0.5 * (hi[k] - lo[k]);
  for (int q = 0; q < nq_box; q++) {
    for (int k = 0; k < dim; k++)
      y1[q * 3 + k] = lo[k] + (box_pts[q * dim + k] + 1.0) * 0.5 *
                                  (hi[k] - lo[k]);
    w1[q] = box_w[q] * jac;
  }
  return nq_box;
}

static void tri_inv(const double *coords, int dim, double *o_v0,
                    double *o_inv) {
  const double *c0 = coords, *c1 = coords + dim, *c2 = coords + 2 * dim;
  double e10 = c1[0] - c0[0];
  double e11 = c1[1] - c0[1];
  double e20 = c2[0] - c0[0];
  double e21 = c2[1] - c0[1];
  double det = e10 * e21 - e11 * e20;
  o_v0[0] = c0[0];
  o_v0[1] = c0[1];
  o_inv[0] = e21 / det;
  o_inv[1] = -e20 / det;
  o_inv[2] = -e11 / det;
  o_inv[3] = e10 / det;
}

/* inverse of the outer tet's edge matrix [e1 e2 e3]: rows (e2 x e3),
 * (e3 x e1), (e1 x e2) over det */
static void tet_inv(const double *coords, double *o_v0, double *o_inv) {
  double e1[3], e2[3], e3[3];
  double det = tet_edges(coords, e1, e2, e3);
  const double *a[3][2] = {{e2, e3}, {e3, e1}, {e1, e2}};
  for (int r = 0; r < 3; r++) {
    const double *u = a[r][0], *v = a[r][1];
    o_inv[3 * r + 0] = (u[1] * v[2] - u[2] * v[1]) / det;
    o_inv[3 * r + 1] = (u[2] * v[0] - u[0] * v[2]) / det;
    o_inv[3 * r + 2] = (u[0] * v[1] - u[1] * v[0]) / det;
  }
  for (int k = 0; k < 3; k++) o_v0[k] = coords[k];
}

static inline void dof_grid(int64_t r, int NX, int NY, int *gx, int *gy,
                            int *gz) {
  *gx = (int)(r % NX);
  int64_t t = r / NX;
  *gy = (int)(t % NY);
  *gz = (int)(t / NY);
}

static void scatter_block(const double *block, int ldb, const int64_t *rows,
                          const int64_t *cols, int nrows, int ncols, int NX,
                          int NY, int K, const int64_t *rowptr,
                          double *vals) {
  for (int i = 0; i < nrows; i++) {
    int rx, ry, rz;
    dof_grid(rows[i], NX, NY, &rx, &ry, &rz);
    int xlo = rx - K; if (xlo < 0) xlo = 0;
    int xhi = rx + K; if (xhi > NX - 1) xhi = NX - 1;
    int Wx = xhi - xlo + 1;
    int ylo = ry - K; if (ylo < 0) ylo = 0;
    int yhi = ry + K; if (yhi > NY - 1) yhi = NY - 1;
    int Wy = yhi - ylo + 1;
    int zlo = rz - K; if (zlo < 0) zlo = 0;
    int64_t base = rowptr[rows[i]];
    for (int j = 0; j < ncols; j++) {
      int cx, cy, cz;
      dof_grid(cols[j], NX, NY, &cx, &cy, &cz);
      int64_t off = ((int64_t)(cz - zlo) * Wy + (cy - ylo)) * Wx + (cx - xlo);
      vals[base + off] += block[i * ldb + j];
    }
  }
}

typedef struct {
  int dim, degree;
  const int8_t *elem_kind;
  const double *elem_coords;
  int nv_max;
  const double *elem_lo, *elem_hi;
  const int64_t *elem_dofs;
  int nloc_max;
  const int64_t *outer_ids;
  int64_t n_outer;
  const int64_t *cand_ptr, *cand_ids;
  const double *box_out_pts, *box_out_w;
  int nq_box_out;
  const double *box_in_pts, *box_in_w;
  int nq_box_in;
  const double *tri_out_pts, *tri_out_w;
  int nq_tri_out;
  const double *tri_in_pts, *tri_in_w;
  int nq_tri_in;
  const double *PHI1_box, *PHI1_tri;
  double delta, eps, cde;
  int L_min, L_max;
  int NX, NY, NZ, K;
  const int64_t *rowptr;
} GeneralArgs;

/* general_core over the outer positions [o_begin, o_end) in blocks of
 * `stride_blk` (for the threaded driver); stride_blk<=0 means contiguous. */
static int64_t general_core_range(const GeneralArgs *a, double *vals,
                                  int64_t *census, int64_t o_first,
                                  int64_t o_step_blk, int64_t blk) {
  int dim = a->dim, degree = a->degree;
  int nl_box = 1;
  for (int k = 0; k < dim; k++) nl_box *= degree + 1;
  int nl_tri = dim == 3 ? 4 : 3 * degree;  /* simplex: tri or tet (P1) */
  int nloc_max = nl_box > nl_tri ? nl_box : nl_tri;
  int nq_max = a->nq_box_in > a->nq_tri_in ? a->nq_box_in : a->nq_tri_in;
  Ctx c;
  c.dim = dim;
  c.degree = degree;
  c.box_pts = a->box_out_pts;
  c.box_w = a->box_out_w;
  c.nq_box = a->nq_box_out;
  c.tri_pts = a->tri_out_pts;
  c.tri_w = a->tri_out_w;
  c.nq_tri = a->nq_tri_out;
  c.delta = a->delta;
  c.eps = a->eps;
  c.cde = a->cde;
  double dm = a->delta - a->eps, dp = a->delta + a->eps;
  c.dme = dm;
  c.dpe = dp;
  c.dm2 = dm * dm;
  c.dp2 = dp * dp;
  c.L_min = a->L_min;
  c.L_max = a->L_max;
  c.census = census;
  int ldb = nloc_max;
  double *b21 = malloc(sizeof(double) * nloc_max * nloc_max);
  double *b22 = malloc(sizeof(double) * nloc_max * nloc_max);
  double *gsum = malloc(sizeof(double) * nq_max);
  double *y1 = malloc(sizeof(double) * nq_max * 3);
  double *w1 = malloc(sizeof(double) * nq_max);
  double (*stack_geo)[12] = malloc(sizeof(double) * 12 * STACK_CAP);
  int *stack_lvl = malloc(sizeof(int) * STACK_CAP);
  double ogeo[12] = {0}, o_lo[3] = {0}, o_hi[3] = {0}, o_v0[3] = {0},
         o_inv[9] = {0}, i_lo[3], i_hi[3];
  int64_t events = 0;
  for (int64_t b0 = o_first; b0 < a->n_outer; b0 += o_step_blk) {
    int64_t b1 = b0 + blk < a->n_outer ? b0 + blk : a->n_outer;
    for (int64_t oi = b0; oi < b1; oi++) {
      int64_t l = a->outer_ids[oi];
      int okind = a->elem_kind[l];
      const double *lc = a->elem_coords + (size_t)l * a->nv_max * dim;
      int nloc2;
      if (okind == 3) {
        for (int t = 0; t < 12; t++) ogeo[t] = lc[t];
        tet_inv(lc, o_v0, o_inv);
        nloc2 = 4;
      } else if (okind == 1) {
        for (int t = 0; t < 3; t++) {
          ogeo[2 * t] = lc[t * dim + 0];
          ogeo[2 * t + 1] = lc[t * dim + 1];
        }
        tri_inv(lc, dim, o_v0, o_inv);
        nloc2 = nl_tri;
      } else {
        for (int k = 0; k < dim; k++) {
          ogeo[k] = a->elem_lo[l * dim + k];
          ogeo[dim + k] = a->elem_hi[l * dim + k];
          o_lo[k] = a->elem_lo[l * dim + k];
          o_hi[k] = a->elem_hi[l * dim + k];
        }
        nloc2 = nl_box;
      }
      for (int64_t ci = a->cand_ptr[oi]; ci < a->cand_ptr[oi + 1]; ci++) {
        int64_t m = a->cand_ids[ci];
        int ikind = a->elem_kind[m];
        for (int k = 0; k < dim; k++) {
          i_lo[k] = a->elem_lo[m * dim + k];
          i_hi[k] = a->elem_hi[m * dim + k];
        }
        const double *PHI1;
        int nloc1, nq1;
        nq1 = inner_data(dim, ikind == 3 ? 3 : (ikind == 1 ? 1 : 0),
                         a->elem_coords + (size_t)m * a->nv_max * dim,
                         a->nv_max, i_lo, i_hi, a->box_in_pts, a->box_in_w,
                         a->nq_box_in, a->tri_in_pts, a->tri_in_w,
                         a->nq_tri_in, y1, w1);
        if (ikind == 1 || ikind == 3) {
          PHI1 = a->PHI1_tri;
          nloc1 = nl_tri;
        } else {
          PHI1 = a->PHI1_box;
          nloc1 = nl_box;
        }
        for (int i = 0; i < nloc1; i++)
          for (int j = 0; j < nloc_max; j++) {
            b21[i * ldb + j] = 0.0;
            b22[i * ldb + j] = 0.0;
          }
        int64_t ev = pair_blocks(&c, okind, ogeo, o_lo, o_hi, o_v0, o_inv,
                                 y1, w1, nq1, PHI1, nloc1, i_lo, i_hi, b21,
                                 b22, ldb, nloc2, gsum, stack_geo, stack_lvl);
        if (ev > 0) {
          events += ev;
          const int64_t *mdofs = a->elem_dofs + (size_t)m * a->nloc_max;
          const int64_t *ldofs = a->elem_dofs + (size_t)l * a->nloc_max;
          scatter_block(b21, ldb, mdofs, ldofs, nloc1, nloc2, a->NX, a->NY,
                        a->K, a->rowptr, vals);
          scatter_block(b22, ldb, mdofs, mdofs, nloc1, nloc1, a->NX, a->NY,
                        a->K, a->rowptr, vals);
        }
      }
    }
  }
  free(b21); free(b22); free(gsum); free(y1); free(w1);
  free(stack_geo); free(stack_lvl);
  return events;
}

#define GENERAL_PARAMS                                                       \
  int dim, int degree, const int8_t *elem_kind, const double *elem_coords,  \
      int nv_max, const double *elem_lo, const double *elem_hi,             \
      const int64_t *elem_dofs, int nloc_max, const int64_t *outer_ids,     \
      int64_t n_outer, const int64_t *cand_ptr, const int64_t *cand_ids,    \
      const double *box_out_pts, const double *box_out_w, int nq_box_out,   \
      const double *box_in_pts, const double *box_in_w, int nq_box_in,      \
      const double *tri_out_pts, const double *tri_out_w, int nq_tri_out,   \
      const double *tri_in_pts, const double *tri_in_w, int nq_tri_in,      \
      const double *PHI1_box, const double *PHI1_tri, double delta,         \
      double eps, double cde, int L_min, int L_max, int NX, int NY, int NZ, \
      int K, const int64_t *rowptr

#define GENERAL_FILL(a)                                                      \
  GeneralArgs a = {dim, degree, elem_kind, elem_coords, nv_max, elem_lo,    \
                   elem_hi, elem_dofs, nloc_max, outer_ids, n_outer,        \
                   cand_ptr, cand_ids, box_out_pts, box_out_w, nq_box_out,  \
                   box_in_pts, box_in_w, nq_box_in, tri_out_pts, tri_out_w, \
                   nq_tri_out, tri_in_pts, tri_in_w, nq_tri_in, PHI1_box,   \
                   PHI1_tri, delta, eps, cde, L_min, L_max, NX, NY, NZ, K,  \
                   rowptr}

/* _general_core (_kernels.py:391-487): accumulates into vals, returns
 * events.  census (nullable, 7 int64): [lvl<Lmax events, Lmax plateau,
 * Lmax dead, Lmax general, point pairs d2<=dm2, shell, skipped]. */
int64_t orc_general_core(GENERAL_PARAMS, double *vals, int64_t *census) {
  GENERAL_FILL(a);
  return general_core_range(&a, vals, census, 0, n_outer > 0 ? n_outer : 1,
                            n_outer > 0 ? n_outer : 1);
}

typedef struct {
  const GeneralArgs *a;
  double *vals;
  int64_t first, step, blk, events;
} ThreadJob;

static void *thread_main(void *p) {
  ThreadJob *j = (ThreadJob *)p;
  j->events = general_core_range(j->a, j->vals, NULL, j->first, j->step,
                                 j->blk);
  return NULL;
}

/* Threaded driver: thread t runs outer blocks t, t+T, t+2T, ... of `blk`
 * outer positions into vals_t[t] (private buffers, or all equal to one
 * shared buffer for timing-only runs).  Returns total events. */
int64_t orc_general_core_mt(GENERAL_PARAMS, double **vals_t, int nthreads,
                            int64_t blk) {
  GENERAL_FILL(a);
  if (nthreads < 1) nthreads = 1;
  if (blk < 1) blk = 1;
  pthread_t *th = malloc(sizeof(pthread_t) * nthreads);
  ThreadJob *jobs = malloc(sizeof(ThreadJob) * nthreads);
  for (int t = 0; t < nthreads; t++) {
    jobs[t].a = &a;
    jobs[t].vals = vals_t[t];
    jobs[t].first = (int64_t)t * blk;
    jobs[t].step = (int64_t)nthreads * blk;
    jobs[t].blk = blk;
    jobs[t].events = 0;
    pthread_create(&th[t], NULL, thread_main, &jobs[t]);
  }
  int64_t ev = 0;
  for (int t = 0; t < nthreads; t++) {
    pthread_join(th[t], NULL);
    ev += jobs[t].events;
  }
  free(th);
  free(jobs);
  return ev;
}

/* _count_candidates / _fill_candidates (_kernels.py:1205-1268).  fill is
 * selected by ids != NULL (then ptr must hold the exclusive scan). */
static void candidates(const int64_t *outer_ids, int64_t n_outer,
                       const int32_t *elem_cell, const double *elem_lo,
                       const double *elem_hi, const uint8_t *inner_mask,
                       const int64_t *cell_ptr, int ncx, int ncy, int ncz,
                       int R, int dim, double dpe, int64_t *counts,
                       const int64_t *ptr, int64_t *ids) {
  for (int64_t oi = 0; oi < n_outer; oi++) {
    int64_t l = outer_ids[oi];
    int c = elem_cell[l];
    int cx = c % ncx, t = c / ncx, cy = t % ncy, cz = t / ncy;
    int zlo = dim == 3 ? (cz - R > 0 ? cz - R : 0) : 0;
    int zhi = dim == 3 ? (cz + R < ncz - 1 ? cz + R : ncz - 1) : 0;
    int ylo = cy - R > 0 ? cy - R : 0, yhi = cy + R < ncy - 1 ? cy + R : ncy - 1;
    int xlo = cx - R > 0 ? cx - R : 0, xhi = cx + R < ncx - 1 ? cx + R : ncx - 1;
    int64_t n = 0;
    int64_t p = ids ? ptr[oi] : 0;
    for (int z2 = zlo; z2 <= zhi; z2++)
      for (int y2 = ylo; y2 <= yhi; y2++)
        for (int x2 = xlo; x2 <= xhi; x2++) {
          int64_t c2 = ((int64_t)z2 * ncy + y2) * ncx + x2;
          for (int64_t e = cell_ptr[c2]; e < cell_ptr[c2 + 1]; e++) {
            if (!inner_mask[e]) continue;
            double gap = 0.0;
            for (int k = 0; k < dim; k++) {
              double d1 = elem_lo[l * dim + k] - elem_hi[e * dim + k];
              double d2 = elem_lo[e * dim + k] - elem_hi[l * dim + k];
              if (d1 > gap) gap = d1;
              if (d2 > gap) gap = d2;
            }
            if (gap < dpe) {
              if (ids)
                ids[p++] = e;
              else
                n++;
            }
          }
        }
    if (!ids) counts[oi] = n;
  }
}

void orc_count_candidates(const int64_t *outer_ids, int64_t n_outer,
                          const int32_t *elem_cell, const double *elem_lo,
                          const double *elem_hi, const uint8_t *inner_mask,
                          const int64_t *cell_ptr, int ncx, int ncy, int ncz,
                          int R, int dim, double dpe, int64_t *counts) {
  candidates(outer_ids, n_outer, elem_cell, elem_lo, elem_hi, inner_mask,
             cell_ptr, ncx, ncy, ncz, R, dim, dpe, counts, NULL, NULL);
}

void orc_fill_candidates(const int64_t *outer_ids, int64_t n_outer,
                         const int32_t *elem_cell, const double *elem_lo,
                         const double *elem_hi, const uint8_t *inner_mask,
                         const int64_t *cell_ptr, int ncx, int ncy, int ncz,
                         int R, int dim, double dpe, const int64_t *ptr,
                         int64_t *ids) {
  candidates(outer_ids, n_outer, elem_cell, elem_lo, elem_hi, inner_mask,
             cell_ptr, ncx, ncy, ncz, R, dim, dpe, NULL, ptr, ids);
}

/* _eidx (_kernels.py:846-868) */
static inline int64_t eidx(int64_t r, int64_t c, int NX, int NY, int K,
                           const int64_t *rowptr) {
  int rx, ry, rz, cx, cy, cz;
  dof_grid(r, NX, NY, &rx, &ry, &rz);
  dof_grid(c, NX, NY, &cx, &cy, &cz);
  int xlo = rx - K; if (xlo < 0) xlo = 0;
  int xhi = rx + K; if (xhi > NX - 1) xhi = NX - 1;
  int Wx = xhi - xlo + 1;
  int ylo = ry - K; if (ylo < 0) ylo = 0;
  int yhi = ry + K; if (yhi > NY - 1) yhi = NY - 1;
  int Wy = yhi - ylo + 1;
  int zlo = rz - K; if (zlo < 0) zlo = 0;
  return rowptr[r] + ((int64_t)(cz - zlo) * Wy + (cy - ylo)) * Wx + (cx - xlo);
}

#define ROW_BOX                                                   \
  int rx, ry, rz;                                                 \
  dof_grid(r, NX, NY, &rx, &ry, &rz);                             \
  int xlo = rx - K > 0 ? rx - K : 0;                              \
  int xhi = rx + K < NX - 1 ? rx + K : NX - 1;                    \
  int ylo = ry - K > 0 ? ry - K : 0;                              \
  int yhi = ry + K < NY - 1 ? ry + K : NY - 1;                    \
  int zlo = rz - K > 0 ? rz - K : 0;                              \
  int zhi = rz + K < NZ - 1 ? rz + K : NZ - 1;

/* _asymmetry_inf (_kernels.py:932-957) */
double orc_asymmetry_inf(const int64_t *rowptr, const double *vals, int NX,
                         int NY, int NZ, int K, int64_t n) {
  double worst = 0.0;
  for (int64_t r = 0; r < n; r++) {
    ROW_BOX
    int64_t p = rowptr[r];
    double rowsum = 0.0;
    for (int cz = zlo; cz <= zhi; cz++)
      for (int cy = ylo; cy <= yhi; cy++)
        for (int cxx = xlo; cxx <= xhi; cxx++) {
          int64_t c = ((int64_t)cz * NY + cy) * NX + cxx;
          int64_t q = eidx(c, r, NX, NY, K, rowptr);
          rowsum += fabs(vals[p] - vals[q]);
          p++;
        }
    if (rowsum > worst) worst = rowsum;
  }
  return worst;
}

/* _matvec (_kernels.py:871-904) */
void orc_matvec(const int64_t *rowptr, const double *vals, const double *x,
                double *y, int NX, int NY, int NZ, int K, int64_t n) {
  for (int64_t r = 0; r < n; r++) {
    ROW_BOX
    double s = 0.0;
    int64_t p = rowptr[r];
    for (int cz = zlo; cz <= zhi; cz++)
      for (int cy = ylo; cy <= yhi; cy++) {
        int64_t base = ((int64_t)cz * NY + cy) * NX + xlo;
        for (int t2 = 0; t2 < xhi - xlo + 1; t2++) s += vals[p++] * x[base + t2];
      }
    y[r] = s;
  }
}

/* _symmetrize (_kernels.py:907-929) */
void orc_symmetrize(const int64_t *rowptr, double *vals, int NX, int NY,
                    int NZ, int K, int64_t n) {
  for (int64_t r = 0; r < n; r++) {
    ROW_BOX
    int64_t p = rowptr[r];
    for (int cz = zlo; cz <= zhi; cz++)
      for (int cy = ylo; cy <= yhi; cy++)
        for (int cxx = xlo; cxx <= xhi; cxx++) {
          int64_t c = ((int64_t)cz * NY + cy) * NX + cxx;
          if (c > r) {
            int64_t q = eidx(c, r, NX, NY, K, rowptr);
            double av = 0.5 * (vals[p] + vals[q]);
            vals[p] = av;
            vals[q] = av;
          }
          p++;
        }
  }
}

/* _diag (_kernels.py:1199-1202) */
void orc_diag(const int64_t *rowptr, const double *vals, int NX, int NY,
              int K, int64_t n, double *out) {
  for (int64_t r = 0; r < n; r++) out[r] = vals[eidx(r, r, NX, NY, K, rowptr)];
}
