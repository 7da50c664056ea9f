// mf_hex.cu -- specialised adaptive assembly for hex Q1 meshes (3D).
//
// Covers BASELINE config #4/#5 stand-ins: pure hex
// mesh, degree 1, tensor outer rule with NO points per axis (2..4), tensor
// inner rule with NI^3 <= 32 points, L_max <= 4.
//
// Work decomposition (one warp per INNER element m of the current colour):
//   lane q1 < NI^3 owns inner quadrature point y_q1 (_inner_data,
//   _kernels.py:316-340) and two accumulators:
//     V[q1][j] = sum over events of this pair of sum_q2 gamma(x_q2, y_q1)
//                w_q2 phi_j(x_q2)                     (reset per pair)
//     G[q1]    = sum over all pairs of sum_j V[q1][j] (= the reference's
//                gsum, since the Q1 shapes sum to one)
//   b21 = -PHI1w^T V is contracted once per pair and A22 once per element
//   (the reference folds both per pair, _kernels.py:139-143, 303-312).
//
// Algorithm 1 (_pair_blocks, _kernels.py:184-313) runs level-synchronously:
// the root sub-cell is classified by every lane, the 8^k children of level
// k are classified one per lane, each child's box recomputed from the root
// along its path with the reference's midpoint arithmetic, so the
// classification is bit-identical.  Events are then integrated by the
// whole warp.  L_max events are split three ways (counted identically):
//   dead    -- exact box gap >= delta+eps: every point pair is skipped by
//              the reference (_kernels.py:134-135); nothing to integrate
//   plateau -- aprx_max < delta-eps: mu == 1 at every point pair, so the
//              event is a rank-1 tensor product (3 x 1D sums)
//   full    -- point pairs evaluated; the outer tensor rule is contracted
//              by sum factorisation (x, then y, then z), 114 DFMA per lane
//              for NO = 3 instead of 27*8.
// Point coordinates and squared distances use the *_rn intrinsics so they
// match the reference bit for bit (eps = 0 ties depend on it).
#include "mf_common.cuh"

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kSplitCap = 64;  // split nodes per level (L_max <= 4)
#ifndef MF_HEX_MINB
#define MF_HEX_MINB 4
#endif

struct Box {
  double lo[3], hi[3];
};

MF_DEV void child_box(const Box &p, int b, Box &c) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double mid = xmul(0.5, xadd(p.lo[k], p.hi[k]));
    if ((b >> k) & 1) {
      c.lo[k] = mid;
      c.hi[k] = p.hi[k];
    } else {
      c.lo[k] = p.lo[k];
      c.hi[k] = mid;
    }
  }
}

// box of the node with path `code` (3 bits per level below the root),
// recomputed from the root with the reference's midpoint arithmetic
MF_DEV Box path_box(const Box &root, uint32_t code, int L) {
  Box g = root;
  for (int l = 2; l <= L; l++) {
    Box c;
    child_box(g, (code >> (3 * (l - 2))) & 7, c);
    g = c;
  }
  return g;
}

enum : int { ACT_NONE = 0, ACT_SPLIT = 1, ACT_UPPER = 2, ACT_PLAT = 3,
             ACT_DEAD = 4, ACT_FULL = 5, ACT_UPPER_FULL = 6 };

// Algorithm-1 decision for one sub-cell (_kernels.py:224-251) plus the
// dead/plateau proofs for L_max events
// Algorithm-1 decision for one sub-cell (_kernels.py:224-251) plus the
// dead/plateau proofs for L_max events.  The proofs use the bounding boxes
// of the quadrature POINT SETS (outer sub-cell points: lo + t_min/max*(hi -
// lo); inner element points: pilo/pihi), which lie strictly inside the
// cells, with a 1e-9 relative margin: every point pair is then certainly
// beyond delta+eps (the reference skips them all, _kernels.py:134-135) or
// certainly inside delta-eps (mu == 1 for all of them).  The event is still
// counted; only its arithmetic changes form.
MF_DEV int classify(const AsmParams &P, const Box &g, int L,
                    const double *ilo, const double *ihi, const double *pilo,
                    const double *pihi, double tmin, double tmax) {
  if (L < P.L_min) return ACT_SPLIT;
  if (L == P.L_max) {
    if (!(aprx_min_d<3>(g.lo, g.hi, ilo, ihi) < P.dpe)) return ACT_NONE;
    if (!P.shortcuts) return ACT_FULL;
    double qlo[3], qhi[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const double w = g.hi[k] - g.lo[k];
      qlo[k] = g.lo[k] + tmin * w;
      qhi[k] = g.lo[k] + tmax * w;
    }
    if (box_dead<3>(P, qlo, qhi, pilo, pihi)) return ACT_DEAD;
    if (aprx_max_sq<3>(qlo, qhi, pilo, pihi) < P.dm2 * (1.0 - 4e-9))
      return ACT_PLAT;
    return ACT_FULL;
  }
  if (aprx_max_lt_dme(P, aprx_max_sq<3>(g.lo, g.hi, ilo, ihi)))
    return P.shortcuts ? ACT_UPPER : ACT_UPPER_FULL;
  if (aprx_min_d<3>(g.lo, g.hi, ilo, ihi) < P.dpe) return ACT_SPLIT;
  return ACT_NONE;
}

// Per-warp uniform state kept in shared memory (not registers) so the
// event code has the register file to itself.
template <int NO>
struct WarpCtx {
  double ilo[3], ihi[3];           // inner element box
  double pilo[3], pihi[3];         // bounding box of its quadrature points
  double olo[3], ohi[3], oinv[3];  // current outer element box
  double blo[33][3], bhi[33][3];   // event boxes of the round (32 = root)
  double X[3][NO];                 // event: outer 1D coordinates
  double sh[3][2][NO];             // event: weighted pullback shapes
};

// Phase 0 of an event: lanes (k, a) compute the outer 1D coordinate
// (exact, like _event_box's x, _kernels.py:115-119) and the two weighted
// pullback shapes (1-s, s) * w_a on axis k; the x axis also carries
// cde * |sub-cell| / 8 / 256.
template <int NO>
MF_DEV void event_axes_to(const AsmParams &P, const double *s_rt,
                          const double *s_rw, WarpCtx<NO> &C, int slot,
                          int lane, double (*X)[NO], double (*sh)[2][NO]) {
  if (lane < 3 * NO) {
    const int k = lane / NO, a = lane - (lane / NO) * NO;
    const double lo = C.blo[slot][k], hi = C.bhi[slot][k];
    double wa = s_rw[a];
    if (k == 0) {
      const double jac = (0.5 * (C.bhi[slot][0] - C.blo[slot][0])) *
                         (0.5 * (C.bhi[slot][1] - C.blo[slot][1])) *
                         (0.5 * (C.bhi[slot][2] - C.blo[slot][2]));
      wa *= P.cde * jac * (1.0 / 256.0);
    }
    const double x = xadd(lo, xmul(s_rt[a], xsub(hi, lo)));
    const double s1 = (x - C.olo[k]) * C.oinv[k];
    X[k][a] = x;
    sh[k][0][a] = (1.0 - s1) * wa;
    sh[k][1][a] = s1 * wa;
  }
}

template <int NO>
MF_DEV void event_axes(const AsmParams &P, const double *s_rt,
                       const double *s_rw, WarpCtx<NO> &C, int slot,
                       int lane) {
  event_axes_to<NO>(P, s_rt, s_rw, C, slot, lane, C.X, C.sh);
  __syncwarp();
}

// mu == 1 at every point pair: V[j] += 256 Sx[jx] Sy[jy] Sz[jz]
template <int NO>
MF_DEV void event_plateau(const AsmParams &P, const double *s_rt,
                          const double *s_rw, WarpCtx<NO> &C, int slot,
                          int lane, double V[8]) {
  event_axes<NO>(P, s_rt, s_rw, C, slot, lane);
  double S[3][2];
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int j = 0; j < 2; j++) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < NO; a++) s += C.sh[k][j][a];
      S[k][j] = s;
    }
  __syncwarp();
#pragma unroll
  for (int jz = 0; jz < 2; jz++)
#pragma unroll
    for (int jy = 0; jy < 2; jy++) {
      const double syz = 256.0 * S[1][jy] * S[2][jz];
#pragma unroll
      for (int jx = 0; jx < 2; jx++)
        V[jx + 2 * jy + 4 * jz] = fma(S[0][jx], syz, V[jx + 2 * jy + 4 * jz]);
    }
}

// Full event: lane q1 evaluates its NO^3 point pairs and contracts them
// by sum factorisation into V.  Every loop is unrolled (x node a, y node b,
// z node c), so the compiler interleaves the NO^3 independent distance /
// mollifier chains of a lane.  Point pairs are classified on the high word
// of the exact d2 (certainly inside delta-eps -> 256, certainly beyond
// delta+eps -> 0, else the shell value).  The shell polynomial is
// evaluated for EVERY point pair, without a warp vote: a vote per (a, b)
// z-line fires on 86% of the lines (some lane of 27 needs the shell there)
// and its branch cost more than the 14% of polynomials it saved (R4-half
// 1300 -> 1275 ms; the straight-line code is what lets the a-unroll pay,
// 1275 -> 1223 ms).  Contraction: z first (2 DFMA per point), then y (4
// per b), then x (8 per a).  Inactive lanes carry a far-away point, so
// every one of their pairs classifies as "beyond".
template <int NO, bool SHARP>
MF_DEV void event_full(const AsmParams &P, const double *s_rt,
                       const double *s_rw, WarpCtx<NO> &C, int slot,
                       const double y[3], int lane, double V[8]) {
  event_axes<NO>(P, s_rt, s_rw, C, slot, lane);
  // the outer y/z weights stay in shared memory (broadcast loads at each
  // use): 24 fewer live registers than register copies
  const double(*shy)[NO] = C.sh[1];
  const double(*shz)[NO] = C.sh[2];
  double sq1[NO], sq2[NO];
#pragma unroll
  for (int b = 0; b < NO; b++) {
    const double d1 = xsub(C.X[1][b], y[1]);
    const double d2 = xsub(C.X[2][b], y[2]);
    sq1[b] = xmul(d1, d1);
    sq2[b] = xmul(d2, d2);
  }
#pragma unroll
  for (int a = 0; a < NO; a++) {
    const double d0 = xsub(C.X[0][a], y[0]);
    const double sq0 = xmul(d0, d0);
    double W[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [jy][jz]
#pragma unroll
    for (int b = 0; b < NO; b++) {
      const double sxy = xadd(sq0, sq1[b]);
      double d2v[NO], mu[NO];
#pragma unroll
      for (int c = 0; c < NO; c++) d2v[c] = xadd(sxy, sq2[c]);
      if (SHARP) {
#pragma unroll
        for (int c = 0; c < NO; c++) mu[c] = d2v[c] < P.dp2 ? 256.0 : 0.0;
      } else {
        double v[NO];
        xi256_fast_n<NO>(P, d2v, v);
#pragma unroll
        for (int c = 0; c < NO; c++) {
          const int hi = __double2hiint(d2v[c]);
          const bool pl = hi < P.hi_dm2;
          const bool sh = !pl && hi <= P.hi_dp2;
          mu[c] = sh ? v[c] : (pl ? 256.0 : 0.0);
        }
      }
      double u0 = 0.0, u1 = 0.0;  // z contraction
#pragma unroll
      for (int c = 0; c < NO; c++) {
        u0 = fma(mu[c], shz[0][c], u0);
        u1 = fma(mu[c], shz[1][c], u1);
      }
#pragma unroll
      for (int jy = 0; jy < 2; jy++) {
        W[jy][0] = fma(u0, shy[jy][b], W[jy][0]);
        W[jy][1] = fma(u1, shy[jy][b], W[jy][1]);
      }
    }
    const double x0 = C.sh[0][0][a], x1 = C.sh[0][1][a];
#pragma unroll
    for (int jz = 0; jz < 2; jz++)
#pragma unroll
      for (int jy = 0; jy < 2; jy++) {
        V[2 * jy + 4 * jz] = fma(x0, W[jy][jz], V[2 * jy + 4 * jz]);
        V[1 + 2 * jy + 4 * jz] = fma(x1, W[jy][jz], V[1 + 2 * jy + 4 * jz]);
      }
  }
  __syncwarp();
}

template <int NO>
MF_DEV void run_full(const AsmParams &P, const double *s_rt,
                     const double *s_rw, WarpCtx<NO> &C, int slot,
                     const double y[3], int lane, double V[8]) {
  if (P.eps == 0.0)
    event_full<NO, true>(P, s_rt, s_rw, C, slot, y, lane, V);
  else
    event_full<NO, false>(P, s_rt, s_rw, C, slot, y, lane, V);
}

template <int NO, int NI>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MF_HEX_MINB)
    k_hex(AsmParams P) {
  constexpr int NQ1 = NI * NI * NI;
  __shared__ double s_phiw[NQ1][8];  // w_ref[q1] * PHI1[q1][i]
  __shared__ double s_phi[NQ1][8];   // PHI1[q1][i]
  __shared__ double s_rt[NO], s_rw[NO];
  __shared__ WarpCtx<NO> s_ctx[kWarpsPerBlock];
  __shared__ double s_buf[kWarpsPerBlock][NQ1][9];
  __shared__ uint32_t s_split[kWarpsPerBlock][2][kSplitCap];

  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * 8; i += blockDim.x) {
    const int q = i / 8, j = i % 8;
    const double ph = Rr.phi_box_in[q * 8 + j];
    s_phi[q][j] = ph;
    s_phiw[q][j] = Rr.box_in_w[q] * ph;
  }
  if (threadIdx.x < NO) {
    s_rt[threadIdx.x] = xmul(xadd(Rr.box_out_x1d[threadIdx.x], 1.0), 0.5);
    s_rw[threadIdx.x] = Rr.box_out_w1d[threadIdx.x];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * kWarpsPerBlock + wib;
  if (t >= P.n_inner) return;
  WarpCtx<NO> &C = s_ctx[wib];
  double(*buf)[9] = s_buf[wib];

  const int64_t m = P.inner[t];
  if (lane < 3) {
    C.ilo[lane] = M.elem_lo[m * 3 + lane];
    C.ihi[lane] = M.elem_hi[m * 3 + lane];
  }
  __syncwarp();
  const double jac_in = (0.5 * (C.ihi[0] - C.ilo[0])) *
                        (0.5 * (C.ihi[1] - C.ilo[1])) *
                        (0.5 * (C.ihi[2] - C.ilo[2]));
  const bool active = lane < NQ1;
  // inactive lanes sit far away: all their pairs classify as "beyond"
  double y[3] = {1e100, 1e100, 1e100};
  if (active) {
#pragma unroll
    for (int k = 0; k < 3; k++)
      y[k] = xadd(C.ilo[k],
                  xmul(xmul(xadd(Rr.box_in_pts[lane * 3 + k], 1.0), 0.5),
                       xsub(C.ihi[k], C.ilo[k])));
  }
  // point-set bounding boxes (outer rule nodes are sorted ascending)
  const double tmin = s_rt[0], tmax = s_rt[NO - 1];
  if (lane < 3) {
    const double w = C.ihi[lane] - C.ilo[lane];
    double pmn = 1e300, pmx = -1e300;
    for (int q = 0; q < NI; q++) {
      const double tq = xmul(xadd(Rr.box_in_x1d[q], 1.0), 0.5);
      pmn = fmin(pmn, C.ilo[lane] + tq * w);
      pmx = fmax(pmx, C.ilo[lane] + tq * w);
    }
    // widen by a relative 1e-12 of the cell so rounding of the points'
    // exact coordinates can never leave the box
    C.pilo[lane] = pmn - 1e-12 * w;
    C.pihi[lane] = pmx + 1e-12 * w;
  }
  __syncwarp();
  double G = 0.0;
  // warp-uniform event counters live in shared memory (lane 0 updates
  // them): 6 fewer registers per lane.  Events = up + plateau + dead + full.
  __shared__ unsigned s_cnt[kWarpsPerBlock][5];
  unsigned *cnt = s_cnt[wib];
  if (lane < 5) cnt[lane] = 0;
  __syncwarp();
#define MF_CNT(k, v)            \
  do {                          \
    if (lane == 0) cnt[k] += (v); \
  } while (0)
  int cx, cy, cz;
  cell_coords(M.elem_cell[m], M.ncx, M.ncy, cx, cy, cz);
  const int Rs = P.R;
  const int xlo = max(cx - Rs, 0), xhi = min(cx + Rs, M.ncx - 1);
  const int ylo = max(cy - Rs, 0), yhi = min(cy + Rs, M.ncy - 1);
  const int zlo = max(cz - Rs, 0), zhi = min(cz + Rs, M.ncz - 1);
  const int nx = xhi - xlo + 1, ny = yhi - ylo + 1;
  const int ncell = nx * ny * (zhi - zlo + 1);
  // this lane's two A21 rows: local DOFs oi and oi + 4 of m (same x/y
  // corner, z and z+1); row box of the implicit pattern per row
  int rx0, ry0, rz0, rz1, rwx, rwy;
  int64_t rb0, rb1;
  {
    const int oi = lane >> 3;
    const int gx = cx + (oi & 1), gy = cy + ((oi >> 1) & 1);
    const int K = P.pat.K;
    rx0 = max(gx - K, 0);
    rwx = min(gx + K, P.pat.NX - 1) - rx0 + 1;
    ry0 = max(gy - K, 0);
    rwy = min(gy + K, P.pat.NY - 1) - ry0 + 1;
    rz0 = max(cz - K, 0);
    rz1 = max(cz + 1 - K, 0);
    const int64_t *md = M.elem_dofs + m * M.nloc_max;
    rb0 = P.pat.rowptr[md[oi]];
    rb1 = P.pat.rowptr[md[oi + 4]];
  }

  for (int base = 0; base < ncell; base += 32) {
    const int ci = base + lane;
    int64_t cand = -1;
    int cpos = 0;  // candidate cell, packed x | y << 10 | z << 20
    if (ci < ncell) {
      const int x2 = xlo + ci % nx;
      const int tt = ci / nx;
      const int y2 = ylo + tt % ny;
      const int z2 = zlo + tt / ny;
      const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
      const int64_t l = M.cell_ptr[c2];
      if (l < M.cell_ptr[c2 + 1] && P.outer_mask[l] &&
          elem_gap<3>(M.elem_lo, M.elem_hi, l, m) < P.dpe) {
        cand = l;
        cpos = x2 | (y2 << 10) | (z2 << 20);
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, cand >= 0);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int64_t l = __shfl_sync(0xffffffffu, cand, src);
      const int lpos = __shfl_sync(0xffffffffu, cpos, src);
      // this lane's two value slots of the pair's A21 block: column DOF oj
      // of l sits at cell(l) + corner offset (hex Q1 DOF grid = vertex
      // grid, fe_space.py:68-80); prefetched into L2 now, written at the
      // end of the pair
      int64_t slot0, slot1;
      {
        const int oj = lane & 7;
        const int gx = (lpos & 1023) + (oj & 1);
        const int gy = ((lpos >> 10) & 1023) + ((oj >> 1) & 1);
        const int gz = (lpos >> 20) + (oj >> 2);
        slot0 = rb0 + ((int64_t)(gz - rz0) * rwy + (gy - ry0)) * rwx +
                (gx - rx0);
        slot1 = rb1 + ((int64_t)(gz - rz1) * rwy + (gy - ry0)) * rwx +
                (gx - rx0);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot0));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot1));
      }
      MF_CNT(0, 1u);
      if (lane < 3) {
        const double lo = M.elem_lo[l * 3 + lane];
        const double hi = M.elem_hi[l * 3 + lane];
        C.olo[lane] = lo;
        C.ohi[lane] = hi;
        C.oinv[lane] = rcp_fast(hi - lo);
        C.blo[32][lane] = lo;
        C.bhi[32][lane] = hi;
      }
      __syncwarp();
      double V[8];
#pragma unroll
      for (int j = 0; j < 8; j++) V[j] = 0.0;
      bool live = false;  // warp-uniform: some plateau/full event
      {
        Box root;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          root.lo[k] = C.olo[k];
          root.hi[k] = C.ohi[k];
        }
        const int act = classify(P, root, 1, C.ilo, C.ihi, C.pilo, C.pihi,
                                 tmin, tmax);
        if (act == ACT_UPPER || act == ACT_PLAT) {
          live = true;
          MF_CNT(act == ACT_UPPER ? 1 : 2, 1u);
          event_plateau<NO>(P, s_rt, s_rw, C, 32, lane, V);
        } else if (act == ACT_FULL || act == ACT_UPPER_FULL) {
          live = true;
          MF_CNT(act == ACT_FULL ? 4 : 1, 1u);
          run_full<NO>(P, s_rt, s_rw, C, 32, y, lane, V);
        } else if (act == ACT_DEAD) {
          MF_CNT(3, 1u);
        } else if (act == ACT_SPLIT) {
          uint32_t *cur = s_split[wib][0], *nxt = s_split[wib][1];
          int nsplit = 1;
          if (lane == 0) cur[0] = 0;
          __syncwarp();
          for (int L = 2; L <= P.L_max && nsplit > 0; L++) {
            const int nchild = nsplit * 8;
            int nnext = 0;
            for (int rb = 0; rb < nchild; rb += 32) {
              const int k = rb + lane;
              int a = ACT_NONE;
              uint32_t code = 0;
              if (k < nchild) {
                code = cur[k >> 3] | ((uint32_t)(k & 7) << (3 * (L - 2)));
                Box rt;
#pragma unroll
                for (int d = 0; d < 3; d++) {
                  rt.lo[d] = C.olo[d];
                  rt.hi[d] = C.ohi[d];
                }
                const Box g = path_box(rt, code, L);
                a = classify(P, g, L, C.ilo, C.ihi, C.pilo, C.pihi, tmin, tmax);
                if (a >= ACT_UPPER && a != ACT_DEAD) {
#pragma unroll
                  for (int d = 0; d < 3; d++) {
                    C.blo[lane][d] = g.lo[d];
                    C.bhi[lane][d] = g.hi[d];
                  }
                }
              }
              const unsigned msplit =
                  __ballot_sync(0xffffffffu, a == ACT_SPLIT);
              if (msplit) {
                const int pos = nnext + __popc(msplit & ((1u << lane) - 1));
                if (a == ACT_SPLIT && pos < kSplitCap) nxt[pos] = code;
                nnext += __popc(msplit);
              }
              const unsigned mplat =
                  __ballot_sync(0xffffffffu, a == ACT_UPPER || a == ACT_PLAT);
              const unsigned mfull = __ballot_sync(
                  0xffffffffu, a == ACT_FULL || a == ACT_UPPER_FULL);
              const unsigned mdead = __ballot_sync(0xffffffffu, a == ACT_DEAD);
              const unsigned mup = __ballot_sync(
                  0xffffffffu, a == ACT_UPPER || a == ACT_UPPER_FULL);
              live |= (mplat | mfull) != 0u;
              if (lane == 0) {
                cnt[3] += __popc(mdead);
                cnt[1] += __popc(mup);
                cnt[2] += __popc(mplat & ~mup);
                cnt[4] += __popc(mfull & ~mup);
              }
              __syncwarp();
              for (unsigned mm = mplat; mm; mm &= mm - 1)
                event_plateau<NO>(P, s_rt, s_rw, C, __ffs(mm) - 1, lane, V);
              for (unsigned mm = mfull; mm; mm &= mm - 1)
                run_full<NO>(P, s_rt, s_rw, C, __ffs(mm) - 1, y, lane, V);
            }
            __syncwarp();
            if (nnext > kSplitCap) {
              // cannot hold the level: flag it (the host raises) rather
              // than return a silently incomplete matrix
              if (lane == 0) atomicAdd(P.counters + MF_CNT_OVERFLOW, 1ull);
              nnext = 0;
            }
            uint32_t *tmp = cur;
            cur = nxt;
            nxt = tmp;
            nsplit = nnext;
          }
        }
      }
      // dead-only pairs have an exactly zero block: skip its contraction
      // and read-modify-write (adding zeros changes no value)
      if (live) {
        // b21[i][j] = -jac_in * sum_q1 phiw[q1][i] V[q1][j]
        if (active) {
#pragma unroll
          for (int j = 0; j < 8; j++) buf[lane][j] = V[j];
        }
        double gs = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) gs += V[j];
        G += gs;
        __syncwarp();
        const int oj = lane & 7, oi = lane >> 3;
        double b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int q = 0; q < NQ1; q++) {
          const double v = buf[q][oj];
          b0 = fma(s_phiw[q][oi], v, b0);
          b1 = fma(s_phiw[q][oi + 4], v, b1);
        }
        __syncwarp();
        const double sc = -P.scale * jac_in;
        // both old values loaded before either store (distinct rows; the
        // compiler cannot prove it and would serialise the two RMWs)
        const double o0 = P.vals[slot0], o1 = P.vals[slot1];
        P.vals[slot0] = o0 + sc * b0;
        P.vals[slot1] = o1 + sc * b1;
      }
    }
  }
  // A22 for the whole element: jac_in * sum_q1 G[q1] phiw[q1][i] phi[q1][j]
  if (active) buf[lane][8] = G;
  __syncwarp();
  const int oj = lane & 7, oi = lane >> 3;
  double b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int q = 0; q < NQ1; q++) {
    const double gq = buf[q][8] * s_phi[q][oj];
    b0 = fma(s_phiw[q][oi], gq, b0);
    b1 = fma(s_phiw[q][oi + 4], gq, b1);
  }
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
  const int64_t col = mdofs[oj];
  const double sc = P.scale * jac_in;
  P.vals[pat_index(P.pat, mdofs[oi], col)] += sc * b0;
  P.vals[pat_index(P.pat, mdofs[oi + 4], col)] += sc * b1;
  if (lane == 0) {
    unsigned long long *Cn = P.counters;
    counter_add(Cn + MF_CNT_EVENTS, (unsigned long long)cnt[1] + cnt[2] +
                                        cnt[3] + cnt[4]);
    counter_add(Cn + MF_CNT_PAIRS, cnt[0]);
    counter_add(Cn + MF_CNT_EV_UPPER, cnt[1]);
    counter_add(Cn + MF_CNT_EV_PLATEAU, cnt[2]);
    counter_add(Cn + MF_CNT_EV_DEAD, cnt[3]);
    counter_add(Cn + MF_CNT_EV_FULL, cnt[4]);
#undef MF_CNT
  }
}

template <int NO, int NI>
cudaError_t launch(const AsmParams &P, cudaStream_t s) {
  const int64_t grid = (P.n_inner + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_hex<NO, NI><<<(unsigned)grid, kWarpsPerBlock * 32, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace

bool mf_hex_supported(const AsmParams &P) {
  const MfMesh &M = P.mesh;
  if (M.dim != 3 || M.degree != 1 || M.nloc_max != 8) return false;
  if (P.L_max > 4) return false;
  // candidate cells are packed x | y << 10 | z << 20 in one register
  if (M.ncx > 1023 || M.ncy > 1023 || M.ncz > 2047) return false;
  const MfRules &R = P.rules;
  if (R.n1d_box_in < 2 || R.n1d_box_in > 3) return false;
  if (R.n1d_box_out < 2 || R.n1d_box_out > 4) return false;
  if (R.nq_box_in != R.n1d_box_in * R.n1d_box_in * R.n1d_box_in) return false;
  if (R.nq_box_out != R.n1d_box_out * R.n1d_box_out * R.n1d_box_out)
    return false;
  return M.kinds_present == 4;  // pure hex (mesh.py:168-178)
}

cudaError_t mf_launch_hex(const AsmParams &P, cudaStream_t s) {
  const int no = P.rules.n1d_box_out, ni = P.rules.n1d_box_in;
  if (ni == 3) {
    if (no == 2) return launch<2, 3>(P, s);
    if (no == 3) return launch<3, 3>(P, s);
    if (no == 4) return launch<4, 3>(P, s);
  } else if (ni == 2) {
    if (no == 2) return launch<2, 2>(P, s);
    if (no == 3) return launch<3, 2>(P, s);
    if (no == 4) return launch<4, 2>(P, s);
  }
  return cudaErrorNotSupported;
}
