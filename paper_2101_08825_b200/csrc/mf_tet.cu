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
// Execution: one thread per (INNER element m of the current colour, stencil
// z-plane) -- 48 colours (cell parity x 6 protos), so same-colour elements
// share no DOF; planes of one parity share no outer vertex (see k_tet), so
// the scatter is race- and atomic-free and deterministic.  Per pair the
// thread walks Algorithm 1 depth first with one geometry per level,
// accumulates V[q1][j] = sum_events sum_q2 gamma w_q2 phi_j(x_q2) and
// contracts it with the inner shapes once per pair; A22 is folded once per
// element from G[q1] = sum_pairs sum_j V[q1][j].  L_max events are split
// into dead / plateau / full like the other kernels; point pairs are
// classified on the high word of the exact d2 with the shell polynomial
// evaluated only when a lane of the warp needs it.
#include "mf_common.cuh"

namespace {

constexpr int kTetLevels = 6;
#ifndef MF_TET_LOADS_FIRST
#define MF_TET_LOADS_FIRST 1
#endif
// loads-first also for larger inner rules (register pressure)
#ifndef MF_TET_LOADS_FIRST_MAXNQ
#define MF_TET_LOADS_FIRST_MAXNQ 11
#endif

// per-thread pair state kept in shared memory, lane-major (stride = block
// size, conflict-free): outer root vertices, the outer inverse map and the
// inner box -- read rarely, so they need not occupy registers
constexpr int kTetThreads = 128;
// Per-rule variants (A/B on the B200, profiles/r2/s4/ab_tet_*.log; all of
// them bit-identical in values and events):
// * lean (inner rules above MF_TET_LEAN_MINNQ points, i.e. tet11): the
//   scatter geometry of the inner element's 4 rows and the G accumulators
//   are not held in registers across the stencil walk.  The row bases and
//   G live in the state rows, the x/y windows are recomputed per live pair
//   (~40 integer instructions against ~5000 per pair).  tet11 spills 96
//   bytes instead of 416: R5-tet-small 1970 -> 1767 ms.  tet4 has no
//   spills to remove and loses L1 to the extra rows (R4-tet 14.96 ->
//   15.04 s), so it keeps the register version.
// * batch (same rules): see bey_row / the root split in k_tet.
// * q2u: outer points of a full event unrolled together; 2 for inner rules
//   of up to 4 points (8 independent mollifier chains, 242 registers, no
//   spills: R4-tet 15.04 -> 14.66 s), 1 for tet11 (2 spills more).
#ifndef MF_TET_LEAN_MINNQ
#define MF_TET_LEAN_MINNQ 5
#endif
#ifndef MF_TET_BATCH_MINNQ
#define MF_TET_BATCH_MINNQ 5
#endif
#ifndef MF_TET_BATCH_HALF_MAXNQ
#define MF_TET_BATCH_HALF_MAXNQ 0
#endif
#ifndef MF_TET_Q2U_MAXNQ
#define MF_TET_Q2U_MAXNQ 4
#endif
template <int NQ1>
struct TetCfg {
  static constexpr bool lean = NQ1 >= MF_TET_LEAN_MINNQ;
  static constexpr bool batch = NQ1 >= MF_TET_BATCH_MINNQ;
  static constexpr int q2u = NQ1 <= MF_TET_Q2U_MAXNQ ? 2 : 1;
  // (A/B knob: the batch in two halves of 4 leaves)
  static constexpr bool batch_half = NQ1 <= MF_TET_BATCH_HALF_MAXNQ;
};
// (tet_state_rows sets the dynamic shared memory per block: 51 KB at 128
// threads for tet4, 72 KB for tet11.  3 blocks/SM lose even without spills
// -- R4-tet 19.6 s, R5-tet-small 4973 ms with the lean state: three blocks
// of state leave no L1 for the coordinate and value gathers.)
// ST_MID: the root's edge midpoints m01 m02 m03 m12 m13 m23, cached when
// the root splits, so a level-2 node is 12 loads instead of 18 midpoint
// computations and a 8-way switch.
// (vertex 0 of the root is rows 0-2 of ST_ROOT; ST_ROWZ and the NQ1 rows of
// ST_G exist for the lean rules only)
// ST_RBOX: the root's vertex box (lo, hi), written when the root splits.
// The vertex box of CORNER child b of Bey's refinement (v_b and the three
// midpoints of its edges) follows from it without min/max: rounding is
// monotone, so min_j rn((v_b + v_j) / 2) = rn((v_b + min_j v_j) / 2), and
// j = b gives v_b itself -- lo = mid(v_b, root lo), hi = mid(v_b, root
// hi), the same bits as the min/max over the child's vertices, in 4
// FP64 instructions per axis instead of 6 compare-and-selects (18
// instructions; ncu: DSETP + FSEL were 20% of k_tet's instructions).
enum : int { ST_ROOT = 0, ST_INV = 12, ST_ILO = 21, ST_IHI = 24, ST_PILO = 27,
             ST_PIHI = 30, ST_MID = 33, ST_RBOX = 51, ST_ROWZ = 57, ST_G = 61 };
// Measured (profiles/r2/s4/ab_tet_cornerbox_*.log, bit-identical): in the
// batched classification (tet11) R5-tet-small 1722 -> 1688 ms; in the
// depth-first walk (tet4) the dynamic child index and the 6 extra state
// rows cost more than the selects saved (R4-tet 14.79 -> 15.07 s), so the
// walk keeps tet_bbox and tet4 has no ST_RBOX rows.
#ifndef MF_TET_CORNER_BOX
#define MF_TET_CORNER_BOX 0
#endif
#ifndef MF_TET_CORNER_BOX_BATCH
#define MF_TET_CORNER_BOX_BATCH 1
#endif
template <int NQ1>
constexpr int tet_state_rows() {
  return TetCfg<NQ1>::lean ? ST_G + NQ1
         : (TetCfg<NQ1>::batch || MF_TET_CORNER_BOX) ? ST_ROWZ
                                                      : ST_RBOX;
}

// cube corners (bit k = axis k) of Kuhn tet p (mesh.py kuhn_corners)
__constant__ int8_t c_tet_corner[6][4] = {{0, 1, 3, 7}, {0, 5, 1, 7},
                                          {0, 3, 2, 7}, {0, 2, 6, 7},
                                          {0, 4, 5, 7}, {0, 6, 4, 7}};

MF_DEV void tet_bbox(const double *g, double *lo, double *hi) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    lo[k] = pmin(g[k], pmin(g[3 + k], pmin(g[6 + k], g[9 + k])));
    hi[k] = pmax(g[k], pmax(g[3 + k], pmax(g[6 + k], g[9 + k])));
  }
}

// child b of parent tet g (exact midpoints, oracle tet_children); written
// with static indices so that g and c stay in registers
MF_DEV void tet_child(const double *g, int b, double *c) {
  double m[6][3];  // m01 m02 m03 m12 m13 m23
#pragma unroll
  for (int k = 0; k < 3; k++) {
    m[0][k] = xmul(0.5, xadd(g[k], g[3 + k]));
    m[1][k] = xmul(0.5, xadd(g[k], g[6 + k]));
    m[2][k] = xmul(0.5, xadd(g[k], g[9 + k]));
    m[3][k] = xmul(0.5, xadd(g[3 + k], g[6 + k]));
    m[4][k] = xmul(0.5, xadd(g[3 + k], g[9 + k]));
    m[5][k] = xmul(0.5, xadd(g[6 + k], g[9 + k]));
  }
#define MF_V(v, src)                               \
  {                                                \
    _Pragma("unroll") for (int k = 0; k < 3; k++) \
      c[3 * (v) + k] = (src)[k];                   \
  }
  switch (b) {
    case 0: MF_V(0, g) MF_V(1, m[0]) MF_V(2, m[1]) MF_V(3, m[2]) break;
    case 1: MF_V(0, m[0]) MF_V(1, g + 3) MF_V(2, m[3]) MF_V(3, m[4]) break;
    case 2: MF_V(0, m[1]) MF_V(1, m[3]) MF_V(2, g + 6) MF_V(3, m[5]) break;
    case 3: MF_V(0, m[2]) MF_V(1, m[4]) MF_V(2, m[5]) MF_V(3, g + 9) break;
    case 4: MF_V(0, m[0]) MF_V(1, m[1]) MF_V(2, m[2]) MF_V(3, m[4]) break;
    case 5: MF_V(0, m[0]) MF_V(1, m[1]) MF_V(2, m[3]) MF_V(3, m[4]) break;
    case 6: MF_V(0, m[1]) MF_V(1, m[2]) MF_V(2, m[4]) MF_V(3, m[5]) break;
    default: MF_V(0, m[1]) MF_V(1, m[3]) MF_V(2, m[4]) MF_V(3, m[5])
  }
#undef MF_V
}

// state rows of the 4 vertices of Bey child b (tet_child's table): root
// vertex i at ST_ROOT + 3 i, edge midpoint j at ST_MID + 3 j
#define MF_M(j) (ST_MID + 3 * (j))
__constant__ int8_t c_bey_row[8][4] = {
    {0, MF_M(0), MF_M(1), MF_M(2)},       {MF_M(0), 3, MF_M(3), MF_M(4)},
    {MF_M(1), MF_M(3), 6, MF_M(5)},       {MF_M(2), MF_M(4), MF_M(5), 9},
    {MF_M(0), MF_M(1), MF_M(2), MF_M(4)}, {MF_M(0), MF_M(1), MF_M(3), MF_M(4)},
    {MF_M(1), MF_M(2), MF_M(4), MF_M(5)}, {MF_M(1), MF_M(3), MF_M(4), MF_M(5)}};
#undef MF_M

// the same table for unrolled code (static shared-memory offsets)
MF_DEV constexpr int bey_row(int b, int v) {
  constexpr int M0 = ST_MID, M1 = ST_MID + 3, M2 = ST_MID + 6,
                M3 = ST_MID + 9, M4 = ST_MID + 12, M5 = ST_MID + 15;
  constexpr int t[8][4] = {{0, M0, M1, M2},   {M0, 3, M3, M4},
                           {M1, M3, 6, M5},   {M2, M4, M5, 9},
                           {M0, M1, M2, M4},  {M0, M1, M3, M4},
                           {M1, M2, M4, M5},  {M1, M3, M4, M5}};
  return t[b][v];
}

// batch: when the root splits and L_max == 2, the 8 leaves are
// classified in one unrolled, branch-free batch (independent chains,
// static state rows), and only the plateau / full leaves are revisited
// (tet11: R5-tet-small 1767 -> 1702 ms.  tet4: 255 registers and 56 bytes
// spilled, R4-tet 15.04 -> 16.02 s, so it keeps the depth-first walk.)

// leaves B0 .. B0+NB-1 of a split root (L_max = 2): event or not, and
// dead / plateau / full by the point-set proofs, as in the walk
template <int B0, int NB>
MF_DEV void tet_classify_leaves(const AsmParams &P, const double *st,
                                double fo, const double *ilo,
                                const double *ihi, const double *plo,
                                const double *phi, unsigned &n_ev,
                                unsigned &m_pl, unsigned &m_full) {
#pragma unroll
  for (int b = B0; b < B0 + NB; b++) {
    double c[12], slo[3], shi[3], qlo[3], qhi[3];
#pragma unroll
    for (int v = 0; v < 4; v++)
#pragma unroll
      for (int k = 0; k < 3; k++)
        c[3 * v + k] = st[(bey_row(b, v) + k) * kTetThreads];
    if (MF_TET_CORNER_BOX_BATCH && b < 4) {
#pragma unroll
      for (int k = 0; k < 3; k++) {
        slo[k] = xmul(0.5, xadd(c[3 * b + k],
                                st[(ST_RBOX + k) * kTetThreads]));
        shi[k] = xmul(0.5, xadd(c[3 * b + k],
                                st[(ST_RBOX + 3 + k) * kTetThreads]));
      }
    } else {
      tet_bbox(c, slo, shi);
    }
    const bool near = aprx_min_d<3>(slo, shi, ilo, ihi) < P.dpe;
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const double cc = 0.25 * ((c[k] + c[3 + k]) + (c[6 + k] + c[9 + k]));
      const double mg = 1e-9 * (shi[k] - slo[k]);
      qlo[k] = cc + fo * (slo[k] - cc) - mg;
      qhi[k] = cc + fo * (shi[k] - cc) + mg;
    }
    const bool dead = box_dead<3>(P, qlo, qhi, plo, phi);
    const bool plat =
        aprx_max_sq<3>(qlo, qhi, plo, phi) < P.dm2 * (1.0 - 4e-9);
    const bool ev_pl = near && !dead && plat;
    const bool ev_fu = near && !dead && !plat;
    n_ev += near ? 1u : 0u;
    m_pl |= (ev_pl ? 1u : 0u) << b;
    m_full |= (ev_fu ? 1u : 0u) << b;
  }
}

// node with path `code` (3 bits per level below the root, L >= 2): the
// level-2 node from the cached root vertices and edge midpoints, deeper
// levels recomputed with exact midpoints
MF_DEV void tet_path(const double *st, uint32_t code, int L, double *g) {
  {
    const int b = code & 7;
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int row = c_bey_row[b][v];
#pragma unroll
      for (int k = 0; k < 3; k++) g[3 * v + k] = st[(row + k) * kTetThreads];
    }
  }
  for (int l = 3; l <= L; l++) {
    double c[12];
    tet_child(g, (code >> (3 * (l - 2))) & 7, c);
#pragma unroll
    for (int u = 0; u < 12; u++) g[u] = c[u];
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
  const double *p;  // &s_state[0][threadIdx.x]
  MF_DEV double v0(int k) const { return p[(ST_ROOT + k) * kTetThreads]; }
  MF_DEV double inv(int k) const { return p[(ST_INV + k) * kTetThreads]; }
};

// mollifier chains written together in a full event
#ifndef MF_TET_CHAINS
#define MF_TET_CHAINS 4
#endif

// full event on sub-tet g (oracle event_tet)
template <int NQO, int NQ1, bool SHARP>
MF_DEV void tet_full(const AsmParams &P, const double *g, const OuterTet &O,
                     const double (*y)[3][32], int lane, const double *s_pts,
                     const double *s_w, double (*V)[4]) {
  double e[3][3];
  const double det = fabs(tet_edges(g, e));
  const double f = det * P.cde * (1.0 / 256.0);
#pragma unroll(TetCfg<NQ1>::q2u)
  for (int q2 = 0; q2 < NQO; q2++) {
    const double p0 = s_pts[3 * q2], p1 = s_pts[3 * q2 + 1],
                 p2 = s_pts[3 * q2 + 2];
    double x[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      if (SHARP)  // eps = 0: the reference's unfused order (ties)
        x[k] = xadd(xadd(xadd(g[k], xmul(p0, e[0][k])), xmul(p1, e[1][k])),
                    xmul(p2, e[2][k]));
      else        // mu is continuous: three FMAs
        x[k] = fma(p2, e[2][k], fma(p1, e[1][k], fma(p0, e[0][k], g[k])));
    }
    const double w2 = s_w[q2] * f;
    const double d0 = x[0] - O.v0(0), d1 = x[1] - O.v0(1),
                 d2 = x[2] - O.v0(2);
    const double rx = O.inv(0) * d0 + O.inv(1) * d1 + O.inv(2) * d2;
    const double ry = O.inv(3) * d0 + O.inv(4) * d1 + O.inv(5) * d2;
    const double rz = O.inv(6) * d0 + O.inv(7) * d1 + O.inv(8) * d2;
    const double s1 = rx * w2, s2 = ry * w2, s3 = rz * w2;
    const double s0 = w2 - s1 - s2 - s3;
    if (SHARP) {
#pragma unroll
      for (int q1 = 0; q1 < NQ1; q1++) {
        const double dx = xsub(x[0], y[q1][0][lane]),
                     dy = xsub(x[1], y[q1][1][lane]),
                     dz = xsub(x[2], y[q1][2][lane]);
        const double dd = xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
        const double mu = dd < P.dp2 ? 256.0 : 0.0;
        V[q1][0] = fma(mu, s0, V[q1][0]);
        V[q1][1] = fma(mu, s1, V[q1][1]);
        V[q1][2] = fma(mu, s2, V[q1][2]);
        V[q1][3] = fma(mu, s3, V[q1][3]);
      }
    } else {
      // eps > 0: mu is continuous, so fused distances and the clamped
      // mollifier (no classification, no vote), contracted at once
      constexpr int GB = MF_TET_CHAINS;
#pragma unroll
      for (int q0 = 0; q0 < NQ1; q0 += GB) {
        double dd[GB], v[GB];
#pragma unroll
        for (int i = 0; i < GB; i++) {
          const int q1 = (q0 + i < NQ1) ? q0 + i : NQ1 - 1;
          const double dx = x[0] - y[q1][0][lane], dy = x[1] - y[q1][1][lane],
                       dz = x[2] - y[q1][2][lane];
          dd[i] = fma(dz, dz, fma(dy, dy, dx * dx));
        }
        // compiler-only barrier: without it the shared-memory point loads
        // of every group are hoisted above the chains and k_tet spills
        // 504 bytes instead of 164 (R4-tet 17.5 -> 23.6 s)
        asm volatile("" ::: "memory");
        xi256_clamped_n<GB>(P, dd, v);
#pragma unroll
        for (int i = 0; i < GB; i++)
          if (q0 + i < NQ1) {
            V[q0 + i][0] = fma(v[i], s0, V[q0 + i][0]);
            V[q0 + i][1] = fma(v[i], s1, V[q0 + i][1]);
            V[q0 + i][2] = fma(v[i], s2, V[q0 + i][2]);
            V[q0 + i][3] = fma(v[i], s3, V[q0 + i][3]);
          }
      }
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
      d[k] = g[k] + p0 * e[0][k] + p1 * e[1][k] + p2 * e[2][k] - O.v0(k);
    const double w2 = s_w[q2] * f;
    const double rx = O.inv(0) * d[0] + O.inv(1) * d[1] + O.inv(2) * d[2];
    const double ry = O.inv(3) * d[0] + O.inv(4) * d[1] + O.inv(5) * d[2];
    const double rz = O.inv(6) * d[0] + O.inv(7) * d[1] + O.inv(8) * d[2];
    SP[0] += w2 * (1.0 - rx - ry - rz);
    SP[1] += w2 * rx;
    SP[2] += w2 * ry;
    SP[3] += w2 * rz;
  }
}

enum : int { ACT_NONE = 0, ACT_SPLIT = 1, ACT_UPPER = 2, ACT_PLAT = 3,
             ACT_DEAD = 4, ACT_FULL = 5 };

// cache operators of the A21 read-modify-writes (A/B knob: 0 default,
// 1 = .cg loads and stores (L2 only), 2 = streaming .cs).  Both lose
// (profiles/r2/s4/ab_tet_valscache_*.log: R4-tet 14.39 -> 15.00 / 14.68 s,
// R5-tet-small 1688 -> 2680 / 1722 ms): the 6 tets of an outer cube share
// corner slots, and those re-reads are the L1 hits.
#ifndef MF_TET_VALS_CACHE
#define MF_TET_VALS_CACHE 0
#endif
#if MF_TET_VALS_CACHE == 1
#define MF_TET_LDV(p) __ldcg(p)
#define MF_TET_STV(p, v) __stcg(p, v)
#elif MF_TET_VALS_CACHE == 2
#define MF_TET_LDV(p) __ldcs(p)
#define MF_TET_STV(p, v) __stcs(p, v)
#else
#define MF_TET_LDV(p) (*(p))
#define MF_TET_STV(p, v) (*(p) = (v))
#endif

// A warp = 32 inner elements (lanes) of the current colour x ONE stencil
// z-plane dz (blockIdx.y); a launch covers the planes of one parity.  The
// lanes walk identical offset sequences (converged on unjittered meshes).
// Same-parity planes are >= 2 cells apart, so their outer tets share no
// vertex: the A21 scatter of one launch is race-free, and the launches run
// in a fixed order (deterministic).  Each warp leaves its per-element G
// partial in gscr[plane][element]; k_tet_a22 sums the planes in order and
// folds A22.  Warps are independent (no block barrier after the start), so
// the short planes at |dz| ~ R do not idle behind the long central ones.
constexpr int kTetWarps = kTetThreads / 32;
// blocks per SM: 2 for every rule (tet4: 235 registers, no spills).  With
// the clamped mollifier the spill-free build wins: R4-tet 17.1 s at 3
// blocks (168 registers, 164 B spilled), 15.7 s at 2, 28.4 s at 4 (128
// registers).  (Round 1, classified mollifier: 3 blocks were faster.)
#ifndef MF_TET_MINB
#ifdef MF_TET_MINB_ALL  // A/B builds: one value for every rule
#define MF_TET_MINB(NQ1) (MF_TET_MINB_ALL)
#else
#define MF_TET_MINB(NQ1) 2
#endif
#endif

template <int NQO, int NQ1>
__global__ void __launch_bounds__(32 * kTetWarps, MF_TET_MINB(NQ1))
    k_tet(AsmParams P, int pass, double *gscr) {
  __shared__ double s_phiw[NQ1][4];
  __shared__ double s_opts[3 * NQO], s_ow[NQO];
  __shared__ double s_y[kTetWarps][NQ1][3][32];  // inner points, lane-major
  extern __shared__ double s_dyn[];  // s_state[tet_state_rows][kTetThreads]
  double(*s_state)[kTetThreads] =
      reinterpret_cast<double(*)[kTetThreads]>(s_dyn);
  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NQ1 * 4; i += blockDim.x) {
    const int q = i / 4, j = i % 4;
    s_phiw[q][j] = Rr.tri_in_w[q] * Rr.phi_tri_in[q * 4 + j];
  }
  for (int i = threadIdx.x; i < NQO; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; k++) s_opts[3 * i + k] = Rr.tri_out_pts[3 * i + k];
    s_ow[i] = Rr.tri_out_w[i];
  }
  // outer rule points lie in the sub-tet shrunk about its centroid by
  // f = 1 - 4 min(barycentric) (their convex hull); + a relative margin
  __shared__ double s_fo;
  if (threadIdx.x == 0) {
    double lmin = 1.0;
    for (int q = 0; q < NQO; q++) {
      const double a = Rr.tri_out_pts[3 * q], b = Rr.tri_out_pts[3 * q + 1],
                   c = Rr.tri_out_pts[3 * q + 2];
      lmin = fmin(lmin, fmin(fmin(a, b), fmin(c, 1.0 - a - b - c)));
    }
    s_fo = fmin(1.0, 1.0 - 4.0 * lmin + 1e-9);
  }
  const int64_t t = ((int64_t)blockIdx.x * kTetWarps + w) * 32 + lane;
  const bool valid = t < P.n_inner;
  const int64_t m = valid ? P.inner[t] : P.inner[0];
  double scale_in;
  {
    const double *c = M.elem_coords + m * M.nv_max * 3;
    double cg[12];
#pragma unroll
    for (int u = 0; u < 12; u++) cg[u] = c[u];
    double e[3][3];
    scale_in = fabs(tet_edges(cg, e));
    // exact inner points (oracle inner_data)
    for (int q = 0; q < NQ1; q++) {
      const double p0 = Rr.tri_in_pts[3 * q], p1 = Rr.tri_in_pts[3 * q + 1],
                   p2 = Rr.tri_in_pts[3 * q + 2];
#pragma unroll
      for (int k = 0; k < 3; k++)
        s_y[w][q][k][lane] = xadd(xadd(xadd(cg[k], xmul(p0, e[0][k])),
                                       xmul(p1, e[1][k])),
                                  xmul(p2, e[2][k]));
    }
  }
  __syncthreads();
  const int Rs = P.R;
  const int pidx = pass + 2 * (int)blockIdx.y;  // plane index dz + R
  const int dz = pidx - Rs;
  if (!valid) return;
  double *st = &s_state[0][threadIdx.x];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double lo = M.elem_lo[m * 3 + k], hi = M.elem_hi[m * 3 + k];
    st[(ST_ILO + k) * kTetThreads] = lo;
    st[(ST_IHI + k) * kTetThreads] = hi;
    // box of the inner rule points, widened by 1e-9 of the element
    double pmn = 1e300, pmx = -1e300;
    for (int q = 0; q < NQ1; q++) {
      pmn = fmin(pmn, s_y[w][q][k][lane]);
      pmx = fmax(pmx, s_y[w][q][k][lane]);
    }
    st[(ST_PILO + k) * kTetThreads] = pmn - 1e-9 * (hi - lo);
    st[(ST_PIHI + k) * kTetThreads] = pmx + 1e-9 * (hi - lo);
  }
  const double fo = s_fo;
  constexpr bool kLean = TetCfg<NQ1>::lean;
  double G[NQ1];  // (lean: unused, the sums live in the ST_G rows)
#pragma unroll
  for (int q = 0; q < NQ1; q++) {
    G[q] = 0.0;
    if constexpr (kLean) st[(ST_G + q) * kTetThreads] = 0.0;
  }
  unsigned c_ev = 0, c_pairs = 0, c_up = 0, c_pl = 0, c_full = 0;
  int cx, cy, cz;
  cell_coords(M.elem_cell[m], M.ncx, M.ncy, cx, cy, cz);
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
  const int z2 = cz + dz;
  if (z2 >= 0 && z2 < M.ncz) {
    // implicit-pattern geometry of this element's 4 rows
    const int tin = (int)(m % 6);
    int64_t rowz[4];
    int rxlo[4], rylo[4], rwx[4], rwy[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int v = c_tet_corner[tin][i];
      const int gx = cx + (v & 1), gy = cy + ((v >> 1) & 1),
                gz = cz + ((v >> 2) & 1);
      rxlo[i] = max(gx - P.pat.K, 0);
      rwx[i] = min(gx + P.pat.K, P.pat.NX - 1) - rxlo[i] + 1;
      rylo[i] = max(gy - P.pat.K, 0);
      rwy[i] = min(gy + P.pat.K, P.pat.NY - 1) - rylo[i] + 1;
      const int rzlo = max(gz - P.pat.K, 0);
      // row base shifted to the z layer of this plane's outer cubes
      rowz[i] = P.pat.rowptr[mdofs[i]] +
                (int64_t)(z2 - rzlo) * rwy[i] * rwx[i];
      if constexpr (kLean)
        st[(ST_ROWZ + i) * kTetThreads] = __longlong_as_double(rowz[i]);
    }
    const double(*y)[3][32] = s_y[w];
    for (int dy = -Rs; dy <= Rs; dy++) {
      const int y2 = cy + dy;
      if (y2 < 0 || y2 >= M.ncy) continue;
      for (int dx = -Rs; dx <= Rs; dx++) {
        const int x2 = cx + dx;
        if (x2 < 0 || x2 >= M.ncx) continue;
        const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
        for (int64_t l = M.cell_ptr[c2]; l < M.cell_ptr[c2 + 1]; l++) {
          if (!P.outer_mask[l]) continue;
          // candidate test (_kernels.py:1225-1233) on the box of l's
          // vertices: elem_lo/hi are exactly their min/max, so this is the
          // same test without two extra gathers
          // (tet11 keeps the elem_lo/hi gathers: its register budget is
          // spent on V[11][4], and the extra live coordinates spill)
          if constexpr (NQ1 > 4) {
            if (!(elem_gap<3>(M.elem_lo, M.elem_hi, l, m) < P.dpe)) continue;
          }
          double g[12];
          {
            const double2 *c2v =
                reinterpret_cast<const double2 *>(M.elem_coords + l * 12);
#pragma unroll
            for (int u = 0; u < 6; u++) {
              const double2 v = c2v[u];
              g[2 * u] = v.x;
              g[2 * u + 1] = v.y;
            }
          }
          if constexpr (NQ1 <= 4) {
            double lo[3], hi[3], gap = 0.0;
            tet_bbox(g, lo, hi);
#pragma unroll
            for (int k = 0; k < 3; k++) {
              const double d1 = xsub(lo[k], st[(ST_IHI + k) * kTetThreads]);
              const double d2 = xsub(st[(ST_ILO + k) * kTetThreads], hi[k]);
              if (d1 > gap) gap = d1;
              if (d2 > gap) gap = d2;
            }
            if (!(gap < P.dpe)) continue;
            // Whole-pair dead proof.  Every descendant of the root lies in
            // its vertex box (Bey midpoints round inside their edge), so
            // (a) if the box's FAR sides are within delta+eps of the inner
            // box on every axis, every descendant passes the _aprx_min
            // test (rounded subtraction is monotone) and none is UPPER:
            // Algorithm 1 splits down to 8^(L_max-1) leaves, and (b) if
            // the box is farther than delta+eps from the inner POINT box,
            // every leaf is dead (its point box lies inside).  The leaves
            // are counted; nothing is integrated (the reference skips
            // every point pair too, _kernels.py:134-135).
            if (P.shortcuts && P.L_max >= 2) {
              bool all = true;
              double sg = 0.0;
#pragma unroll
              for (int k = 0; k < 3; k++) {
                all = all &&
                      xsub(hi[k], st[(ST_IHI + k) * kTetThreads]) < P.dpe &&
                      xsub(st[(ST_ILO + k) * kTetThreads], lo[k]) < P.dpe;
                const double mg = 1e-9 * (hi[k] - lo[k]);
                const double gk =
                    pmax(pmax(lo[k] - mg - st[(ST_PIHI + k) * kTetThreads],
                              st[(ST_PILO + k) * kTetThreads] - hi[k] - mg),
                         0.0);
                sg += gk * gk;
              }
              if (all && sg >= P.dp2 * (1.0 + 2e-9)) {
                const unsigned nleaf = 1u << (3 * (P.L_max - 1));
                c_pairs++;
                c_ev += nleaf;
                continue;
              }
            }
          }
          c_pairs++;
          const int tout = (int)(l % 6);
          const OuterTet O{st};
          {
#pragma unroll
            for (int u = 0; u < 12; u++) st[(ST_ROOT + u) * kTetThreads] = g[u];
            double e[3][3];
            const double det = tet_edges(g, e);
            const double idet = rcp_fast(det);
            // rows (e2 x e3), (e3 x e1), (e1 x e2) over det (oracle tet_inv)
#pragma unroll
            for (int r = 0; r < 3; r++) {
              const double *u = e[(r + 1) % 3], *v = e[(r + 2) % 3];
              st[(ST_INV + 3 * r + 0) * kTetThreads] =
                  (u[1] * v[2] - u[2] * v[1]) * idet;
              st[(ST_INV + 3 * r + 1) * kTetThreads] =
                  (u[2] * v[0] - u[0] * v[2]) * idet;
              st[(ST_INV + 3 * r + 2) * kTetThreads] =
                  (u[0] * v[1] - u[1] * v[0]) * idet;
            }
          }
          double V[NQ1][4];
#pragma unroll
          for (int q = 0; q < NQ1; q++)
#pragma unroll
            for (int j = 0; j < 4; j++) V[q][j] = 0.0;
          double SP[4] = {0.0, 0.0, 0.0, 0.0};
          unsigned ev = 0;
          bool live = false;  // some plateau/full event: nonzero block
          // Algorithm 1, depth first over a path code (3 bits per level
          // below the root); the node is recomputed from the root
          uint32_t code = 0;
          int L = 1;
          for (;;) {
            double slo[3], shi[3], ilo[3], ihi[3];
            if (MF_TET_CORNER_BOX && L == 2 && (code & 4) == 0) {
              const int b = code & 3;  // corner child: see ST_RBOX
#pragma unroll
              for (int k = 0; k < 3; k++) {
                const double vb = st[(ST_ROOT + 3 * b + k) * kTetThreads];
                slo[k] = xmul(0.5, xadd(vb, st[(ST_RBOX + k) * kTetThreads]));
                shi[k] =
                    xmul(0.5, xadd(vb, st[(ST_RBOX + 3 + k) * kTetThreads]));
              }
            } else {
              tet_bbox(g, slo, shi);
            }
#pragma unroll
            for (int k = 0; k < 3; k++) {
              ilo[k] = st[(ST_ILO + k) * kTetThreads];
              ihi[k] = st[(ST_IHI + k) * kTetThreads];
            }
            int act = ACT_NONE;
            if (L < P.L_min) {
              act = ACT_SPLIT;
            } else if (L == P.L_max) {
              if (aprx_min_d<3>(slo, shi, ilo, ihi) < P.dpe) {
                if (!P.shortcuts) {
                  act = ACT_FULL;
                } else {
                  // dead / plateau proofs on the point-set boxes (see
                  // mf_hex.cu classify): every point pair certainly beyond
                  // delta+eps, or certainly inside delta-eps
                  double qlo[3], qhi[3], plo[3], phi[3];
#pragma unroll
                  for (int k = 0; k < 3; k++) {
                    const double c =
                        0.25 * ((g[k] + g[3 + k]) + (g[6 + k] + g[9 + k]));
                    const double mg = 1e-9 * (shi[k] - slo[k]);
                    qlo[k] = c + fo * (slo[k] - c) - mg;
                    qhi[k] = c + fo * (shi[k] - c) + mg;
                    plo[k] = st[(ST_PILO + k) * kTetThreads];
                    phi[k] = st[(ST_PIHI + k) * kTetThreads];
                  }
                  if (box_dead<3>(P, qlo, qhi, plo, phi))
                    act = ACT_DEAD;
                  else if (aprx_max_sq<3>(qlo, qhi, plo, phi) <
                           P.dm2 * (1.0 - 4e-9))
                    act = ACT_PLAT;
                  else
                    act = ACT_FULL;
                }
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
              if (act == ACT_PLAT) c_pl++;
              if (act == ACT_FULL) c_full++;
              const bool plateau =
                  act == ACT_PLAT || (act == ACT_UPPER && P.shortcuts);
              const bool full =
                  act == ACT_FULL || (act == ACT_UPPER && !P.shortcuts);
              live |= plateau || full;
              if (plateau)
                tet_plateau<NQO>(P, g, O, s_opts, s_ow, SP);
              else if (full && P.eps > 0.0)
                tet_full<NQO, NQ1, false>(P, g, O, y, lane, s_opts, s_ow, V);
              else if (full)
                tet_full<NQO, NQ1, true>(P, g, O, y, lane, s_opts, s_ow, V);
            }
            if (act == ACT_SPLIT) {
              if (L == 1) {
                // the root splits: cache its edge midpoints (exact, as
                // tet_child computes them) for every level-2 node; the
                // first child is (v0, m01, m02, m03)
#pragma unroll
                for (int k = 0; k < 3; k++) {
                  if constexpr (TetCfg<NQ1>::batch || MF_TET_CORNER_BOX) {
                    st[(ST_RBOX + k) * kTetThreads] = slo[k];
                    st[(ST_RBOX + 3 + k) * kTetThreads] = shi[k];
                  }
                  const double m01 = xmul(0.5, xadd(g[k], g[3 + k]));
                  const double m02 = xmul(0.5, xadd(g[k], g[6 + k]));
                  const double m03 = xmul(0.5, xadd(g[k], g[9 + k]));
                  st[(ST_MID + 9 + k) * kTetThreads] =
                      xmul(0.5, xadd(g[3 + k], g[6 + k]));
                  st[(ST_MID + 12 + k) * kTetThreads] =
                      xmul(0.5, xadd(g[3 + k], g[9 + k]));
                  st[(ST_MID + 15 + k) * kTetThreads] =
                      xmul(0.5, xadd(g[6 + k], g[9 + k]));
                  st[(ST_MID + k) * kTetThreads] = m01;
                  st[(ST_MID + 3 + k) * kTetThreads] = m02;
                  st[(ST_MID + 6 + k) * kTetThreads] = m03;
                  g[3 + k] = m01;
                  g[6 + k] = m02;
                  g[9 + k] = m03;
                }
                if (TetCfg<NQ1>::batch && P.L_max == 2 && P.shortcuts) {
                  double ilo[3], ihi[3], plo[3], phi[3];
#pragma unroll
                  for (int k = 0; k < 3; k++) {
                    ilo[k] = st[(ST_ILO + k) * kTetThreads];
                    ihi[k] = st[(ST_IHI + k) * kTetThreads];
                    plo[k] = st[(ST_PILO + k) * kTetThreads];
                    phi[k] = st[(ST_PIHI + k) * kTetThreads];
                  }
                  unsigned m_pl = 0, m_full = 0, n_ev = 0;
                  if constexpr (TetCfg<NQ1>::batch_half) {
                    tet_classify_leaves<0, 4>(P, st, fo, ilo, ihi, plo, phi,
                                              n_ev, m_pl, m_full);
                    asm volatile("" ::: "memory");
                    tet_classify_leaves<4, 4>(P, st, fo, ilo, ihi, plo, phi,
                                              n_ev, m_pl, m_full);
                  } else {
                    tet_classify_leaves<0, 8>(P, st, fo, ilo, ihi, plo, phi,
                                              n_ev, m_pl, m_full);
                  }
                  ev += n_ev;
                  c_pl += __popc(m_pl);
                  c_full += __popc(m_full);
                  unsigned todo = m_pl | m_full;
                  live |= todo != 0;
                  while (todo) {
                    const int b = __ffs(todo) - 1;
                    todo &= todo - 1;
                    tet_path(st, (uint32_t)b, 2, g);
                    if ((m_pl >> b) & 1)
                      tet_plateau<NQO>(P, g, O, s_opts, s_ow, SP);
                    else if (P.eps > 0.0)
                      tet_full<NQO, NQ1, false>(P, g, O, y, lane, s_opts, s_ow,
                                                V);
                    else
                      tet_full<NQO, NQ1, true>(P, g, O, y, lane, s_opts, s_ow,
                                               V);
                  }
                  break;
                }
                L = 2;
                continue;
              }
              ++L;  // first child: code bits of level L stay 0
              double c[12];
              tet_child(g, 0, c);
#pragma unroll
              for (int u = 0; u < 12; u++) g[u] = c[u];
              continue;
            }
            // next sibling, climbing while the current level is exhausted
            while (L > 1 && ((code >> (3 * (L - 2))) & 7) == 7) {
              code &= ~(7u << (3 * (L - 2)));
              --L;
            }
            if (L == 1) break;
            code += 1u << (3 * (L - 2));
            tet_path(st, code, L, g);
          }
          c_ev += ev;
          // dead-only pairs have an exactly zero block: adding it would
          // change no value, so the 16 read-modify-writes are skipped
          if (live) {
            double spsum = (SP[0] + SP[1]) + (SP[2] + SP[3]);
            const double sc = -P.scale * scale_in;
            if constexpr (kLean) {
              // (the values computed above are dead across the walk)
#pragma unroll
              for (int i = 0; i < 4; i++) {
                const int v = c_tet_corner[tin][i];
                const int gx = cx + (v & 1), gy = cy + ((v >> 1) & 1);
                rxlo[i] = max(gx - P.pat.K, 0);
                rwx[i] = min(gx + P.pat.K, P.pat.NX - 1) - rxlo[i] + 1;
                rylo[i] = max(gy - P.pat.K, 0);
                rwy[i] = min(gy + P.pat.K, P.pat.NY - 1) - rylo[i] + 1;
                rowz[i] =
                    __double_as_longlong(st[(ST_ROWZ + i) * kTetThreads]);
              }
            }
#if MF_TET_LOADS_FIRST
            // the 16 old values are loaded together before any store, so
            // their latencies overlap (the compiler cannot hoist them past
            // the stores itself: it cannot prove the slots distinct)
            double old[4][4];
            if constexpr (NQ1 <= MF_TET_LOADS_FIRST_MAXNQ) {
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const int v = c_tet_corner[tout][j];
                const int gx = x2 + (v & 1), gy = y2 + ((v >> 1) & 1),
                          gzo = (v >> 2) & 1;
#pragma unroll
                for (int i = 0; i < 4; i++)
                  old[i][j] = MF_TET_LDV(
                      P.vals + rowz[i] +
                      ((int64_t)gzo * rwy[i] + (gy - rylo[i])) * rwx[i] +
                      (gx - rxlo[i]));
              }
            }
#endif
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
                          gzo = (v >> 2) & 1;
                const int64_t slot =
                    rowz[i] +
                    ((int64_t)gzo * rwy[i] + (gy - rylo[i])) * rwx[i] +
                    (gx - rxlo[i]);
#if MF_TET_LOADS_FIRST
                if constexpr (NQ1 <= MF_TET_LOADS_FIRST_MAXNQ)
                  MF_TET_STV(P.vals + slot, old[i][j] + sc * b);
                else
                  P.vals[slot] += sc * b;
#else
                P.vals[slot] += sc * b;
#endif
              }
            }
#pragma unroll
            for (int q = 0; q < NQ1; q++) {
              double s = spsum;
#pragma unroll
              for (int j = 0; j < 4; j++) s += V[q][j];
              if constexpr (kLean)
                st[(ST_G + q) * kTetThreads] += s;
              else
                G[q] += s;
            }
          }
        }
      }
    }
  }
  double *gp = gscr + ((int64_t)pidx * P.n_inner + t) * NQ1;
#pragma unroll
  for (int q = 0; q < NQ1; q++)
    gp[q] = kLean ? st[(ST_G + q) * kTetThreads] : G[q];
  const unsigned mask = __activemask();
  // every event is upper, plateau, dead or full
  const unsigned c_dead = c_ev - c_up - c_pl - c_full;
  const unsigned v[6] = {c_ev, c_pairs, c_up, c_pl, c_dead, c_full};
  const int slot[6] = {MF_CNT_EVENTS, MF_CNT_PAIRS, MF_CNT_EV_UPPER,
                       MF_CNT_EV_PLATEAU, MF_CNT_EV_DEAD, MF_CNT_EV_FULL};
  const bool leader = lane == __ffs(mask) - 1;
#pragma unroll
  for (int k = 0; k < 6; k++) {
    const unsigned s = __reduce_add_sync(mask, v[k]);
    if (leader && s) atomicAdd(P.counters + slot[k], (unsigned long long)s);
  }
}

// A22 of each element from the plane partials of G, summed in plane order
template <int NQ1>
__global__ void __launch_bounds__(128) k_tet_a22(AsmParams P,
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
  double cg[12];
  const double *c = M.elem_coords + m * M.nv_max * 3;
#pragma unroll
  for (int u = 0; u < 12; u++) cg[u] = c[u];
  double e[3][3];
  const double sc = P.scale * fabs(tet_edges(cg, e));
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t r = mdofs[i];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      double b = 0.0;
#pragma unroll
      for (int q = 0; q < NQ1; q++)
        b = fma(Gt[q] * (Rr.tri_in_w[q] * Rr.phi_tri_in[q * 4 + i]),
                Rr.phi_tri_in[q * 4 + j], b);
      P.vals[pat_index(P.pat, r, mdofs[j])] += sc * b;
    }
  }
}

// (A/B knob: an explicit minimal shared-memory carve-out changes nothing,
// R4-tet 14381.6 vs 14382.5 ms, profiles/r2/s4/ab_tet_carveout_*.log: the
// driver already picks the smallest carve-out that holds 2 blocks.)
#ifndef MF_TET_CARVEOUT
#define MF_TET_CARVEOUT 0
#endif

template <int NQO, int NQ1>
cudaError_t launch(const AsmParams &P, double *gscr, cudaStream_t s) {
  const unsigned gx = (unsigned)((P.n_inner + 32 * kTetWarps - 1) /
                                 (32 * kTetWarps));
  const size_t dyn = sizeof(double) * tet_state_rows<NQ1>() * kTetThreads;
  cudaError_t ea = cudaFuncSetAttribute(
      k_tet<NQO, NQ1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (ea != cudaSuccess) return ea;
#if MF_TET_CARVEOUT
  {
    // shared-memory carve-out: just enough for the 2 resident blocks, the
    // rest of the 256 KB stays L1 for the coordinate and value gathers
    cudaFuncAttributes fa;
    ea = cudaFuncGetAttributes(&fa, k_tet<NQO, NQ1>);
    if (ea != cudaSuccess) return ea;
    const size_t need = 2 * (dyn + fa.sharedSizeBytes + 1024);
    int pct = (int)((need * 100 + 228 * 1024 - 1) / (228 * 1024));
    if (pct > 100) pct = 100;
    ea = cudaFuncSetAttribute(k_tet<NQO, NQ1>,
                              cudaFuncAttributePreferredSharedMemoryCarveout,
                              pct);
    if (ea != cudaSuccess) return ea;
  }
#endif
  for (int pass = 0; pass < 2; pass++) {
    const int planes = pass == 0 ? P.R + 1 : P.R;
    if (planes < 1) continue;
    k_tet<NQO, NQ1><<<dim3(gx, planes), kTetThreads, dyn, s>>>(P, pass,
                                                                gscr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_tet_a22<NQ1><<<(unsigned)((P.n_inner + 127) / 128), 128, 0, s>>>(P,
                                                                    gscr);
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

size_t mf_tet_scratch_doubles(const AsmParams &P, int64_t n_colour_max) {
  return (size_t)(2 * P.R + 1) * (size_t)n_colour_max *
         (size_t)P.rules.nq_tri_in;
}

cudaError_t mf_launch_tet(const AsmParams &P, double *gscr, cudaStream_t s) {
  const int no = P.rules.nq_tri_out, ni = P.rules.nq_tri_in;
#define MF_T(NO_, NI_) \
  if (no == NO_ && ni == NI_) return launch<NO_, NI_>(P, gscr, s);
  MF_T(1, 1) MF_T(4, 1) MF_T(11, 1)
  MF_T(1, 4) MF_T(4, 4) MF_T(11, 4)
  MF_T(1, 11) MF_T(4, 11) MF_T(11, 11)
#undef MF_T
  return cudaErrorNotSupported;
}
