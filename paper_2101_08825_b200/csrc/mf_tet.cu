// mf_tet.cu -- adaptive assembly for P1 tetrahedral meshes (new element).
//
// BASELINE configs #4/#5 as written: the 6-tet (Kuhn) split of a cube grid,
// optionally with jittered vertices (mesh.py build_mesh(kind="tet")).  The
// reference has no tetrahedra; this kernel extends its
// Algorithm 1 in the same style and is checked against the C restatement
// in oracle/mf_oracle.c (event_tet, tet_children, tet_inv):
//   * sub-cells are tets (4 vertices); the Algorithm-1 distances use the
//     bounding box of the sub-tet's vertices against the inner element box,
//     as the reference does for triangles (_kernels.py:214-222);
//   * a split makes the 8 children of Bey's red refinement, vertices by
//     exact midpoint arithmetic;
//   * an event maps the simplex outer rule affinely onto the sub-tet,
//     weights times |det|, shapes by pulling back through the outer
//     element's inverse map (the reference's _event_tri in 3D).
//
// Execution follows mf_2d.cu: one thread per INNER element m of the
// current colour (48 colours: cell parity x 6 protos, so same-colour
// elements share no DOF and the scatter is race- and atomic-free).  Per
// pair the thread walks Algorithm 1 depth first with one geometry per
// level, accumulates V[q1][j] = sum_events sum_q2 gamma w_q2 phi_j(x_q2) and
// contracts it with the inner shapes once per pair; A22 is folded once per
// element from G[q1] = sum_pairs sum_j V[q1][j].  L_max events are split
// into dead / plateau / full like the other kernels; point pairs are
// classified on the high word of the exact d2 with the shell polynomial
// evaluated only when a lane of the warp needs it.
#include "mf_common.cuh"

namespace {

constexpr int kTetLevels = 6;

// cube corners (bit k = axis k) of Kuhn tet p (mesh.py kuhn_corners)
__constant__ int8_t c_tet_corner[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7},
                                          {0, 3, 2, 7}, {0, 2, 6, 7},
                                          {0, 4, 5, 7}, {0, 6, 4, 7}};
// children of the red refinement over {x0..x3, m01, m02, m03, m12, m13, m23}
__constant__ int8_t c_tet_child[8][4] = {{0, 4, 5, 6}, {4, 1, 7, 8},
                                         {5, 7, 2, 9}, {6, 8, 9, 3},
                                         {4, 5, 6, 8}, {4, 5, 7, 8},
                                         {5, 6, 8, 9}, {5, 7, 8, 9}};
__constant__ int8_t c_tet_edge[6][2] = {{0, 1}, {0, 2}, {0, 3},
                                        {1, 2}, {1, 3}, {2, 3}};

MF_DEV void tet_bbox(const double *g, double *lo, double *hi) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = pmin(g[k], pmin(g[3 + k], pmin(g[6 + k], g[9 + k])));
    hi[k] = pmax(g[k], pmax(g[3 + k], pmax(g[6 + k], g[9 + k])));
  }
}

// vertex v of child b of parent tet g (exact midpoints, mf_oracle.c)
MF_DEV void tet_child(const double *g, int b, double *c) {
#pragma unroll
  for (int v = 0; v < 4; v++) {
    const int p = c_tet_child[b][v];
    if (p < 4) {
#pragma unroll
      for (int k = 0; k < 3; k++) c[3 * v + k] = g[3 * p + k];
    } else {
      const int a = c_tet_edge[p - 4][0], e = c_tet_edge[p - 4][1];
#pragma unroll
      for (int k = 0; k < 3; k++)
        c[3 * v + k] = xmul(0.5, xadd(g[3 * a + k], g[3 * e + k]));
    }
  }
}

// edges from vertex 0 (exact) and |det| (rounding-level, weights only)
MF_DEV double tet_edges(const double *g, double (*e)[3]) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    e[0][k] = xsub(g[3 + k], g[k]);
    e[1][k] = xsub(g[6 + k], g[k]);
    e[2][k] = xsub(g[9 + k], g[k]);
  }
  const double c0 = e[1][1] * e[2][2] - e[1][2] * e[2][1];
  const double c1 = e[1][2] * e[2][0] - e[1][0] * e[2][2];
  const double c2 = e[1][0] * e[2][1] - e[1][1] * e[2][0];
  return (e[0][0] * c0 + e[0][1] * c1) + e[0][2] * c2;
}

struct OuterTet {
  double v0[3], inv[9];
};

// full event on sub-tet g (oracle event_tet)
template <int NQO, int NQ1, bool SHARP>
MF_DEV void tet_full(const AsmParams &P, const double *g, const OuterTet &O,
                     const double (*y)[3], const double *s_pts,
                     const double *s_w, double (*V)[4]) {
  double e[3][3];
  const double det = fabs(tet_edges(g, e));
  const double f = det * P.cde * (1.0 / 256.0);
#pragma unroll 1
  for (int q2 = 0; q2 < NQO; q2++) {
    const double p0 = s_pts[3 * q2], p1 = s_pts[3 * q2 + 1],
                 p2 = s_pts[3 * q2 + 2];
    double x[3];
#pragma unroll
    for (int k = 0; k < 3; k++)
      x[k] = xadd(xadd(xadd(g[k], xmul(p0, e[0][k])), xmul(p1, e[1][k])),
                  xmul(p2, e[2][k]));
    const double w2 = s_w[q2] * f;
    const double d0 = x[0] - O.v0[0], d1 = x[1] - O.v0[1], d2 = x[2] - O.v0[2];
    const double rx = O.inv[0] * d0 + O.inv[1] * d1 + O.inv[2] * d2;
    const double ry = O.inv[3] * d0 + O.inv[4] * d1 + O.inv[5] * d2;
    const double rz = O.inv[6] * d0 + O.inv[7] * d1 + O.inv[8] * d2;
    const double s1 = rx * w2, s2 = ry * w2, s3 = rz * w2;
    const double s0 = w2 - s1 - s2 - s3;
    double mu[NQ1];
    bool anysh = false;
    unsigned shm = 0;
#pragma unroll
    for (int q1 = 0; q1 < NQ1; q1++) {
      const double dx = xsub(x[0], y[q1][0]), dy = xsub(x[1], y[q1][1]),
                   dz = xsub(x[2], y[q1][2]);
      const double dd = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
      if (SHARP) {
        mu[q1] = dd < P.dp2 ? 256.0 : 0.0;
      } else {
        const int hi = __double2hiint(dd);
        const bool pl = hi < P.hi_dm2, sk = hi > P.hi_dp2;
        const bool sh = !(pl || sk);
        mu[q1] = sh ? dd : (pl ? 256.0 : 0.0);
        shm |= (unsigned)sh << q1;
        anysh |= sh;
      }
    }
    if (!SHARP && __any_sync(__activemask(), anysh)) {
#pragma unroll
      for (int q1 = 0; q1 < NQ1; q1++) {
        const double v = xi256_unclamped(P, mu[q1]);
        if ((shm >> q1) & 1u) mu[q1] = v;
      }
    }
#pragma unroll
    for (int q1 = 0; q1 < NQ1; q1++) {
      V[q1][0] = fma(mu[q1], s0, V[q1][0]);
      V[q1][1] = fma(mu[q1], s1, V[q1][1]);
      V[q1][2] = fma(mu[q1], s2, V[q1][2]);
      V[q1][3] = fma(mu[q1], s3, V[q1][3]);
    }
  }
}

// mu == 1 at every point pair: SP[j] += cde sum_q2 w_q2 phi_j(x_q2)
template <int NQO>
MF_DEV void tet_plateau(const AsmParams &P, const double *g,
                        const OuterTet &O, const double *s_pts,
                        const double *s_w, double *SP) {
  double e[3][3];
  const double f = fabs(tet_edges(g, e)) * P.cde;
#pragma unroll 1
  for (int q2 = 0; q2 < NQO; q2++) {
    const double p0 = s_pts[3 * q2], p1 = s_pts[3 * q2 + 1],
                 p2 = s_pts[3 * q2 + 2];
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; k++)
      d[k] = g[k] + p0 * e[0][k] + p1 * e[1][k] + p2 * e[2][k] - O.v0[k];
    const double w2 = s_w[q2] * f;
    const double rx = O.inv[0] * d[0] + O.inv[1] * d[1] + O.inv[2] * d[2];
    const double ry = O.inv[3] * d[0] + O.inv[4] * d[1] + O.inv[5] * d[2];
    const double rz = O.inv[6] * d[0] + O.inv[7] * d[1] + O.inv[8] * d[2];
    SP[0] += w2 * (1.0 - rx - ry - rz);
    SP[1] += w2 * rx;
    SP[2] += w2 * ry;
    SP[3] += w2 * rz;
  }
}

enum : int { ACT_NONE = 0, ACT_SPLIT = 1, ACT_UPPER = 2, ACT_PLAT = 3,
             ACT_DEAD = 4, ACT_FULL = 5 };

template <int NQO, int NQ1>
__global__ void __launch_bounds__(128, 2) k_tet(AsmParams P) {
  __shared__ double s_phiw[NQ1][4], s_phi[NQ1][4];
  __shared__ double s_opts[3 * NQO], s_ow[NQO];
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * 4; i += blockDim.x) {
    const int q = i / 4, j = i % 4;
    const double ph = Rr.phi_tri_in[q * 4 + j];
    s_phi[q][j] = ph;
    s_phiw[q][j] = Rr.tri_in_w[q] * ph;
  }
  for (int i = threadIdx.x; i < NQO; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; k++) s_opts[3 * i + k] = Rr.tri_out_pts[3 * i + k];
    s_ow[i] = Rr.tri_out_w[i];
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.n_inner) return;
  const int64_t m = P.inner[t];

  // inner element: exact points (oracle inner_data) and |det|
  double y[NQ1][3];
  double ilo[3], ihi[3], scale_in;
  {
    const double *c = M.elem_coords + m * M.nv_max * 3;
    double cg[12];
#pragma unroll
    for (int u = 0; u < 12; u++) cg[u] = c[u];
    double e[3][3];
    scale_in = fabs(tet_edges(cg, e));
#pragma unroll
    for (int q = 0; q < NQ1; q++) {
      const double p0 = Rr.tri_in_pts[3 * q], p1 = Rr.tri_in_pts[3 * q + 1],
                   p2 = Rr.tri_in_pts[3 * q + 2];
#pragma unroll
      for (int k = 0; k < 3; k++)
        y[q][k] = xadd(xadd(xadd(cg[k], xmul(p0, e[0][k])),
                            xmul(p1, e[1][k])),
                       xmul(p2, e[2][k]));
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {
      ilo[k] = M.elem_lo[m * 3 + k];
      ihi[k] = M.elem_hi[m * 3 + k];
    }
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
  // implicit-pattern geometry of this element's 4 rows
  const int tin = (int)(m % 6);
  int64_t rowbase[4];
  int rxlo[4], rylo[4], rzlo[4], rwx[4], rwy[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int v = c_tet_corner[tin][i];
    const int gx = cx + (v & 1), gy = cy + ((v >> 1) & 1),
              gz = cz + ((v >> 2) & 1);
    rxlo[i] = max(gx - P.pat.K, 0);
    rwx[i] = min(gx + P.pat.K, P.pat.NX - 1) - rxlo[i] + 1;
    rylo[i] = max(gy - P.pat.K, 0);
    rwy[i] = min(gy + P.pat.K, P.pat.NY - 1) - rylo[i] + 1;
    rzlo[i] = max(gz - P.pat.K, 0);
    rowbase[i] = P.pat.rowptr[mdofs[i]];
  }

  for (int dz = -Rs; dz <= Rs; dz++) {
    const int z2 = cz + dz;
    if (z2 < 0 || z2 >= M.ncz) continue;
    for (int dy = -Rs; dy <= Rs; dy++) {
      const int y2 = cy + dy;
      if (y2 < 0 || y2 >= M.ncy) continue;
      for (int dx = -Rs; dx <= Rs; dx++) {
        const int x2 = cx + dx;
        if (x2 < 0 || x2 >= M.ncx) continue;
        const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
        for (int64_t l = M.cell_ptr[c2]; l < M.cell_ptr[c2 + 1]; l++) {
          if (!P.outer_mask[l]) continue;
          if (!(elem_gap<3>(M.elem_lo, M.elem_hi, l, m) < P.dpe)) continue;
          c_pairs++;
          const int tout = (int)(l % 6);
          OuterTet O;
          double root[12];
          {
            const double *c = M.elem_coords + l * M.nv_max * 3;
#pragma unroll
            for (int u = 0; u < 12; u++) root[u] = c[u];
            double e[3][3];
            const double det = tet_edges(root, e);
            const double idet = rcp_fast(det);
            // rows (e2 x e3), (e3 x e1), (e1 x e2) over det (oracle tet_inv)
#pragma unroll
            for (int r = 0; r < 3; r++) {
              const double *u = e[(r + 1) % 3], *v = e[(r + 2) % 3];
              O.inv[3 * r + 0] = (u[1] * v[2] - u[2] * v[1]) * idet;
              O.inv[3 * r + 1] = (u[2] * v[0] - u[0] * v[2]) * idet;
              O.inv[3 * r + 2] = (u[0] * v[1] - u[1] * v[0]) * idet;
            }
#pragma unroll
            for (int k = 0; k < 3; k++) O.v0[k] = root[k];
          }
          double V[NQ1][4];
#pragma unroll
          for (int q = 0; q < NQ1; q++)
#pragma unroll
            for (int j = 0; j < 4; j++) V[q][j] = 0.0;
          double SP[4] = {0.0, 0.0, 0.0, 0.0};
          unsigned long long ev = 0;
          double geo[kTetLevels + 1][12];
          int child[kTetLevels + 1];
#pragma unroll
          for (int u = 0; u < 12; u++) geo[1][u] = root[u];
          int L = 1;
          for (;;) {
            double slo[3], shi[3];
            tet_bbox(geo[L], slo, shi);
            int act = ACT_NONE;
            if (L < P.L_min) {
              act = ACT_SPLIT;
            } else if (L == P.L_max) {
              if (aprx_min_d<3>(slo, shi, ilo, ihi) < P.dpe) {
                if (!P.shortcuts)
                  act = ACT_FULL;
                else if (box_dead<3>(P, slo, shi, ilo, ihi))
                  act = ACT_DEAD;
                else if (aprx_max_lt_dme(P, aprx_max_sq<3>(slo, shi, ilo,
                                                           ihi)))
                  act = ACT_PLAT;
                else
                  act = ACT_FULL;
              }
            } else if (aprx_max_lt_dme(P,
                                       aprx_max_sq<3>(slo, shi, ilo, ihi))) {
              act = ACT_UPPER;
            } else if (aprx_min_d<3>(slo, shi, ilo, ihi) < P.dpe) {
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
              if (plateau)
                tet_plateau<NQO>(P, geo[L], O, s_opts, s_ow, SP);
              else if (full && P.eps > 0.0)
                tet_full<NQO, NQ1, false>(P, geo[L], O, y, s_opts, s_ow, V);
              else if (full)
                tet_full<NQO, NQ1, true>(P, geo[L], O, y, s_opts, s_ow, V);
            }
            if (act == ACT_SPLIT) {
              ++L;
              child[L] = 0;
              tet_child(geo[L - 1], 0, geo[L]);
              continue;
            }
            bool done = false;
            for (;;) {
              if (L == 1) {
                done = true;
                break;
              }
              if (++child[L] < 8) {
                tet_child(geo[L - 1], child[L], geo[L]);
                break;
              }
              --L;
            }
            if (done) break;
          }
          if (ev) {
            c_ev += ev;
            double spsum = (SP[0] + SP[1]) + (SP[2] + SP[3]);
            const double sc = -P.scale * scale_in;
#pragma unroll
            for (int i = 0; i < 4; i++) {
              double mi = 0.0;
#pragma unroll
              for (int q = 0; q < NQ1; q++) mi += s_phiw[q][i];
#pragma unroll
              for (int j = 0; j < 4; j++) {
                double b = mi * SP[j];
#pragma unroll
                for (int q = 0; q < NQ1; q++) b = fma(s_phiw[q][i], V[q][j], b);
                const int v = c_tet_corner[tout][j];
                const int gx = x2 + (v & 1), gy = y2 + ((v >> 1) & 1),
                          gz = z2 + ((v >> 2) & 1);
                const int64_t slot =
                    rowbase[i] +
                    ((int64_t)(gz - rzlo[i]) * rwy[i] + (gy - rylo[i])) *
                        rwx[i] +
                    (gx - rxlo[i]);
                P.vals[slot] += sc * b;
              }
            }
#pragma unroll
            for (int q = 0; q < NQ1; q++) {
              double s = spsum;
#pragma unroll
              for (int j = 0; j < 4; j++) s += V[q][j];
              G[q] += s;
            }
          }
        }
      }
    }
  }
  // A22 of the element
  const double sc = P.scale * scale_in;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t r = mdofs[i];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      double b = 0.0;
#pragma unroll
      for (int q = 0; q < NQ1; q++)
        b = fma(G[q] * s_phiw[q][i], s_phi[q][j], b);
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

template <int NQO, int NQ1>
cudaError_t launch(const AsmParams &P, cudaStream_t s) {
  const int block = 128;
  const int64_t grid = (P.n_inner + block - 1) / block;
  k_tet<NQO, NQ1><<<(unsigned)grid, block, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace

bool mf_tet_supported(const AsmParams &P) {
  const MfMesh &M = P.mesh;
  if (M.dim != 3 || M.degree != 1 || M.kinds_present != 8) return false;
  if (M.nloc_max != 4 || M.nv_max != 4 || P.L_max > kTetLevels) return false;
  const int no = P.rules.nq_tri_out, ni = P.rules.nq_tri_in;
  return (no == 1 || no == 4 || no == 11) && (ni == 1 || ni == 4 || ni == 11);
}

cudaError_t mf_launch_tet(const AsmParams &P, cudaStream_t s) {
  const int no = P.rules.nq_tri_out, ni = P.rules.nq_tri_in;
#define MF_T(NO_, NI_) \
  if (no == NO_ && ni == NI_) return launch<NO_, NI_>(P, s);
  MF_T(1, 1) MF_T(4, 1) MF_T(11, 1)
  MF_T(1, 4) MF_T(4, 4) MF_T(11, 4)
  MF_T(1, 11) MF_T(4, 11) MF_T(11, 11)
#undef MF_T
  return cudaErrorNotSupported;
}
