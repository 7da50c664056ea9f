// mf_hex2.cu -- hex Q1 assembly kernel for L_max == 2 with eps > 0 and
// the shortcuts on (the BASELINE #4/#5 stand-ins R4/R5).
//
// Same work decomposition and results as k_hex (mf_hex.cu: one warp per
// inner element, lane = inner quadrature point, colour-scheduled
// scatter), restructured around what L_max == 2 makes separable:
//
// * The root sub-cell and its 8 children are axis-aligned boxes built
//   from 3 intervals per axis (lower half, upper half, whole).  Every
//   Algorithm-1 quantity is a max or an ordered sum of per-axis terms
//   (_aprx_min / _aprx_max, _kernels.py:80-102), so 9 lanes compute the
//   per-(axis, interval) terms once per pair with the reference's exact
//   arithmetic, and 9 lanes (8 children + root) combine three of them
//   each: one classification pass per pair instead of a root pass, a
//   child pass and a path-box recomputation.
// * The outer quadrature coordinates and weighted pullback shapes of an
//   event are per-axis too: the same 9 lanes compute them once per pair
//   for all 8 children (k_hex: once per event).
// * Plateau events (mu == 1 at every point pair) add the same rank-1
//   term to every inner point, so they are folded into the pair's block
//   through sum_q1 phiw[q1][i] instead of through V.
// * Full events evaluate the mollifier on coordinates scaled by 1/eps:
//   q = |x - y|^2 / eps^2 has its high word clamped to the shell
//   [(alpha-1)^2, (alpha+1)^2] with integer min/max (xi(+-1) = 256 / 0 and
//   four vanishing derivatives there make the 2^-20 slack invisible,
//   < 1e-21), one MUFU rsqrt seed z, and the Newton step folded into
//     2 r = 2 alpha - W (3 - W z),  W = q z
//   (3 DP operations; same 1.5 e^2 error as k_hex's 5-operation form),
//   then the degree-9 xi in 2 r: 9 DP operations per point pair, no
//   selects, no integer fix-ups.
// * Measured on B200: the kernel is dispatch-bound.  FP64 and integer-ALU
//   instructions occupy an SM sub-partition's dispatch port for 2 cycles,
//   everything else for 1; 2 (FP64 + ALU) + rest reproduces the SM active
//   cycles of the ncu capture to 0.3%.  More warps or more interleaved
//   chains change nothing (measured); only fewer instructions do.
// * The candidate boxes of a 32-cell batch are staged in shared memory by
//   the lanes that found them, so a pair starts without a global load.
//
// Events are counted exactly as the reference does (same aprx_min /
// aprx_max decisions, bit for bit); dead / plateau / full only choose the
// form of the arithmetic.
#include "mf_common.cuh"

namespace {

#ifndef MF_HEX2_WARPS
#define MF_HEX2_WARPS 1
#endif
#ifndef MF_HEX2_MINB
#define MF_HEX2_MINB 20
#endif
constexpr int kWarps2 = MF_HEX2_WARPS;

template <int NO>
struct Ctx2 {
  double ilo[3], ihi[3];    // inner element box
  double pilo[3], pihi[3];  // bounding box of its quadrature points
  double box[32][6];        // candidate boxes of the batch (lo[3], hi[3])
  double X[9][NO];          // (axis, interval): outer coordinates / eps
  double sh[9][2][NO];      // weighted pullback shapes (jacobian folded in)
  double S[9][2];           // their sums over the rule
  double jac_in;            // inner jacobian
  long long rb[32][2];      // per lane: value base of its two A21 rows
  int rbox[32][6];          // per lane: row box x0, y0, z0, z1, wx, wy
};

// 256 xi((delta - d)/eps) from N scaled squared distances q = d^2/eps^2,
// written stage by stage so the N chains interleave.  With the MUFU seed
// z ~ 1/sqrt(q):  W = q z,  T = 3 - W z,  rho = 2 alpha - W T = 2 r  (the
// Newton step for sqrt(q) with every constant folded: 3 DP operations, no
// integer exponent fix-up), then xi as a polynomial in rho = 2 r (the
// coefficients 315/2, -420/8, 378/32, -180/128, 35/512 are exact).
// (Dropping one clamp side for events proven to have no point pair beyond
// delta+eps, or none inside delta-eps, was measured: 860.6 vs 855.4 ms on
// R4-half with four event instantiations -- no gain, not kept.)
template <int N>
MF_DEV void xi256_scaled_n(const AsmParams &P, const double *q, double *out) {
  double qc[N], z[N], W[N], T[N], r[N], r2[N], p[N];
#pragma unroll
  for (int i = 0; i < N; i++) {
    int hi = __double2hiint(q[i]);
    hi = min(max(hi, P.hq_lo), P.hq_hi);
    qc[i] = __hiloint2double(hi, __double2loint(q[i]));
  }
#pragma unroll
  for (int i = 0; i < N; i++)
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(z[i]) : "d"(qc[i]));
#pragma unroll
  for (int i = 0; i < N; i++) W[i] = qc[i] * z[i];
#pragma unroll
  for (int i = 0; i < N; i++) T[i] = fma(-W[i], z[i], 3.0);
#pragma unroll
  for (int i = 0; i < N; i++) r[i] = fma(-W[i], T[i], P.alpha2);
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

// Full event of child (hx, hy, hz): lane q1 evaluates its NO^3 point pairs
// and contracts them by sum factorisation (z, then y, then x) into V.
template <int NO>
MF_DEV void event_full2(const AsmParams &P, const Ctx2<NO> &C, int ix, int iy,
                        int iz, const double ys[3], double V[8]) {
  const double *Xx = C.X[ix], *Xy = C.X[iy], *Xz = C.X[iz];
  const double(*shx)[NO] = C.sh[ix];
  const double(*shy)[NO] = C.sh[iy];
  const double(*shz)[NO] = C.sh[iz];
  double sq1[NO], sq2[NO];
#pragma unroll
  for (int b = 0; b < NO; b++) {
    const double d1 = Xy[b] - ys[1];
    const double d2 = Xz[b] - ys[2];
    sq1[b] = d1 * d1;
    sq2[b] = d2 * d2;
  }
#pragma unroll
  for (int a = 0; a < NO; a++) {
    const double d0 = Xx[a] - ys[0];
    double W[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [jy][jz]
#pragma unroll
    for (int b = 0; b < NO; b++) {
      const double sxy = fma(d0, d0, sq1[b]);
      double qq[NO], mu[NO];
#pragma unroll
      for (int c = 0; c < NO; c++) qq[c] = sxy + sq2[c];
      xi256_scaled_n<NO>(P, qq, mu);
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
    const double x0 = shx[0][a], x1 = shx[1][a];
#pragma unroll
    for (int jz = 0; jz < 2; jz++)
#pragma unroll
      for (int jy = 0; jy < 2; jy++) {
        V[2 * jy + 4 * jz] = fma(x0, W[jy][jz], V[2 * jy + 4 * jz]);
        V[1 + 2 * jy + 4 * jz] = fma(x1, W[jy][jz], V[1 + 2 * jy + 4 * jz]);
      }
  }
}

template <int NO, int NI>
__global__ void __launch_bounds__(kWarps2 * 32, MF_HEX2_MINB)
    k_hex2(AsmParams P) {
  constexpr int NQ1 = NI * NI * NI;
  __shared__ double2 s_phiw2[NQ1][4];  // w_ref[q1] * PHI1[q1][i], [i + 4]
  __shared__ double s_phi[NQ1][8];     // PHI1[q1][i]
  __shared__ double s_pw[8];           // sum_q1 w_ref[q1] PHI1[q1][i]
  __shared__ double s_rt[NO], s_rw[NO];
  __shared__ Ctx2<NO> s_ctx[kWarps2];
  __shared__ double s_buf[kWarps2][NQ1][9];
  __shared__ unsigned s_cnt[kWarps2][5];

  const MfMesh &M = P.mesh;
  const MfRules &Rr = P.rules;
  for (int i = threadIdx.x; i < NQ1 * 8; i += blockDim.x) {
    const int q = i / 8, j = i % 8;
    const double ph = Rr.phi_box_in[q * 8 + j];
    s_phi[q][j] = ph;
    const double pw = Rr.box_in_w[q] * ph;
    if (j < 4)
      s_phiw2[q][j].x = pw;
    else
      s_phiw2[q][j - 4].y = pw;
  }
  if (threadIdx.x < NO) {
    s_rt[threadIdx.x] = xmul(xadd(Rr.box_out_x1d[threadIdx.x], 1.0), 0.5);
    s_rw[threadIdx.x] = Rr.box_out_w1d[threadIdx.x];
  }
  if (threadIdx.x >= 8 && threadIdx.x < 16) {
    const int j = threadIdx.x - 8;
    double s = 0.0;
    for (int q = 0; q < NQ1; q++)
      s += Rr.box_in_w[q] * Rr.phi_box_in[q * 8 + j];
    s_pw[j] = s;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * kWarps2 + wib;
  if (t >= P.n_inner) return;
  Ctx2<NO> &C = s_ctx[wib];
  double(*buf)[9] = s_buf[wib];
  unsigned *cnt = s_cnt[wib];

  const int64_t m = P.inner[t];
  if (lane < 3) {
    C.ilo[lane] = M.elem_lo[m * 3 + lane];
    C.ihi[lane] = M.elem_hi[m * 3 + lane];
  }
  if (lane < 5) cnt[lane] = 0;
  __syncwarp();
  if (lane == 0)
    C.jac_in = (0.5 * (C.ihi[0] - C.ilo[0])) * (0.5 * (C.ihi[1] - C.ilo[1])) *
               (0.5 * (C.ihi[2] - C.ilo[2]));
  const bool active = lane < NQ1;
  // this lane's inner point, scaled by 1/eps; inactive lanes mirror a
  // real point (their results are never read)
  double ys[3];
  {
    const int pq = lane % NQ1;
#pragma unroll
    for (int k = 0; k < 3; k++)
      ys[k] = P.inv_eps *
              xadd(C.ilo[k],
                   xmul(xmul(xadd(Rr.box_in_pts[pq * 3 + k], 1.0), 0.5),
                        xsub(C.ihi[k], C.ilo[k])));
  }
  // point-set bounding boxes (outer rule nodes are sorted ascending)
  if (lane < 3) {
    const double w = C.ihi[lane] - C.ilo[lane];
    double pmn = 1e300, pmx = -1e300;
    for (int q = 0; q < NI; q++) {
      const double tq = xmul(xadd(Rr.box_in_x1d[q], 1.0), 0.5);
      pmn = fmin(pmn, C.ilo[lane] + tq * w);
      pmx = fmax(pmx, C.ilo[lane] + tq * w);
    }
    // widened by a relative 1e-12 of the cell: rounding of the points'
    // exact coordinates can never leave the box
    C.pilo[lane] = pmn - 1e-12 * w;
    C.pihi[lane] = pmx + 1e-12 * w;
  }
  if (active) buf[lane][8] = 0.0;  // G: sum over all pairs of sum_j V[j]
  __syncwarp();
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
  const int oj = lane & 7, oi = lane >> 3;
  {
    const int gx = cx + (oi & 1), gy = cy + ((oi >> 1) & 1);
    const int K = P.pat.K;
    const int rx0 = max(gx - K, 0), ry0 = max(gy - K, 0);
    C.rbox[lane][0] = rx0;
    C.rbox[lane][1] = ry0;
    C.rbox[lane][2] = max(cz - K, 0);
    C.rbox[lane][3] = max(cz + 1 - K, 0);
    C.rbox[lane][4] = min(gx + K, P.pat.NX - 1) - rx0 + 1;
    C.rbox[lane][5] = min(gy + K, P.pat.NY - 1) - ry0 + 1;
    const int64_t *md = M.elem_dofs + m * M.nloc_max;
    C.rb[lane][0] = P.pat.rowptr[md[oi]];
    C.rb[lane][1] = P.pat.rowptr[md[oi + 4]];
  }
  __syncwarp();
  const double dead2 = P.dp2 * (1.0 + 1e-9), plat2 = P.dm2 * (1.0 - 4e-9);

  for (int base = 0; base < ncell; base += 32) {
    // ---- scan: every lane looks at one stencil cell, and classifies the
    // pair it finds there all by itself (root + 8 children) ----
    const int ci = base + lane;
    bool cand = false;
    int cpos = 0;       // candidate cell, packed x | y << 10 | z << 20
    unsigned cls = 0u;  // bits 0-7 full children, 8-15 plateau children,
                        // 16 root plateau (UPPER)
    unsigned ndead = 0u;
    if (ci < ncell) {
      const int x2 = xlo + ci % nx;
      const int tt = ci / nx;
      const int y2 = ylo + tt % ny;
      const int z2 = zlo + tt / ny;
      const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
      const int64_t l = M.cell_ptr[c2];
      if (l < M.cell_ptr[c2 + 1] && P.outer_mask[l]) {
        // per axis: root gap (the candidate test of _count_candidates,
        // _kernels.py:1225-1233, is the root's _aprx_min), root max
        // separation, and for the two halves the gap test and the
        // point-set terms of the dead / plateau proofs
        double gap = 0.0, smx[3], pd[3][2], pp[3][2];
        unsigned alive = 0u;  // bit 2k + h: half h of axis k within reach
#pragma unroll
        for (int k = 0; k < 3; k++) {
          const double olo = M.elem_lo[l * 3 + k], ohi = M.elem_hi[l * 3 + k];
          C.box[lane][k] = olo;
          C.box[lane][3 + k] = ohi;
          const double ilo = C.ilo[k], ihi = C.ihi[k];
          const double r1 = xsub(olo, ihi), r2 = xsub(ilo, ohi);
          if (r1 > gap) gap = r1;
          if (r2 > gap) gap = r2;
          const double ra = xmul(r1, r1), rb = xmul(r2, r2);
          smx[k] = (ra > rb) ? ra : rb;
          const double mid = xmul(0.5, xadd(olo, ohi));  // _kernels.py:262
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const double lo = h ? mid : olo, hi = h ? ohi : mid;
            const double d1 = xsub(lo, ihi), d2 = xsub(ilo, hi);
            // _aprx_min term max(0, d1, d2) < dpe
            if (d1 < P.dpe && d2 < P.dpe) alive |= 1u << (2 * k + h);
            const double w = hi - lo;
            const double qlo = lo + s_rt[0] * w, qhi = lo + s_rt[NO - 1] * w;
            const double e1 = qlo - C.pihi[k], e2 = C.pilo[k] - qhi;
            const double gd = pmax(pmax(e1, e2), 0.0);
            pd[k][h] = gd * gd;
            pp[k][h] = pmax(e1 * e1, e2 * e2);
          }
        }
        if (gap < P.dpe) {
          cand = true;
          cpos = x2 | (y2 << 10) | (z2 << 20);
          bool split = true;
          if (P.L_min <= 1) {
            const double sm = xadd(xadd(smx[0], smx[1]), smx[2]);
            if (aprx_max_lt_dme(P, sm)) {  // root inside delta - eps
              split = false;
              cls = 1u << 16;
            }
          }
          if (split) {
#pragma unroll
            for (int c = 0; c < 8; c++) {
              const int hx = c & 1, hy = (c >> 1) & 1, hz = c >> 2;
              const unsigned need =
                  (1u << hx) | (4u << hy) | (16u << hz);
              if ((alive & need) == need) {
                const double sd = pd[0][hx] + pd[1][hy] + pd[2][hz];
                const double sp = pp[0][hx] + pp[1][hy] + pp[2][hz];
                if (sd >= dead2)
                  ndead++;
                else if (sp < plat2)
                  cls |= 0x100u << c;
                else
                  cls |= 1u << c;
              }
            }
          }
        }
      }
    }
    // live pairs only enter the pair loop; the counters take everything
    unsigned mask = __ballot_sync(0xffffffffu, cls != 0u);
    {
      const unsigned mc = __ballot_sync(0xffffffffu, cand);
      const unsigned mu = __ballot_sync(0xffffffffu, (cls >> 16) != 0u);
      const unsigned packed = ndead | (__popc(cls & 0xffu) << 10) |
                              (__popc(cls & 0xff00u) << 20);
      const unsigned tot = __reduce_add_sync(0xffffffffu, packed);
      if (lane == 0) {
        cnt[0] += __popc(mc);
        cnt[1] += __popc(mu);
        cnt[2] += tot >> 20;
        cnt[3] += tot & 1023u;
        cnt[4] += (tot >> 10) & 1023u;
      }
    }
    __syncwarp();
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int lpos = __shfl_sync(0xffffffffu, cpos, src);
      const unsigned pcls = __shfl_sync(0xffffffffu, cls, src);
      const unsigned mfull = pcls & 0xffu;
      const unsigned mplat = (pcls >> 8) & 0x1ffu;  // bit 8 = the root
      // this lane's two value slots of the pair's A21 block: column DOF oj
      // of l sits at cell(l) + corner offset (hex Q1 DOF grid = vertex
      // grid, fe_space.py:68-80); prefetched into L2 now, written at the
      // end of the pair
      int64_t slot0, slot1;
      {
        const int gx = (lpos & 1023) + (oj & 1);
        const int gy = ((lpos >> 10) & 1023) + ((oj >> 1) & 1);
        const int gz = (lpos >> 20) + (oj >> 2);
        const int *rbx = C.rbox[lane];
        const int rwx = rbx[4], rwy = rbx[5];
        const int xy = (gy - rbx[1]) * rwx + (gx - rbx[0]);
        slot0 = C.rb[lane][0] + (int64_t)(gz - rbx[2]) * (rwy * rwx) + xy;
        slot1 = C.rb[lane][1] + (int64_t)(gz - rbx[3]) * (rwy * rwx) + xy;
#ifndef MF_HEX2_NOPF
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot0));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.vals + slot1));
#endif
      }
      // ---- event axes of the pair: lanes (axis k, interval h) ----
      if (lane < 9) {
        const int k = lane / 3, h = lane - 3 * (lane / 3);
        const double olo = C.box[src][k], ohi = C.box[src][3 + k];
        const double mid = xmul(0.5, xadd(olo, ohi));
        const double lo = (h == 1) ? mid : olo;
        const double hi = (h == 0) ? mid : ohi;
        const double oinv = rcp_fast(ohi - olo);
        double hw = 0.5 * (hi - lo);
        if (k == 0) hw *= P.cde * (1.0 / 256.0);
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int q = 0; q < NO; q++) {
          const double x = xadd(lo, xmul(s_rt[q], xsub(hi, lo)));
          const double sx = (x - olo) * oinv;
          const double wa = s_rw[q] * hw;
          const double f0 = (1.0 - sx) * wa, f1 = sx * wa;
          C.X[lane][q] = x * P.inv_eps;
          C.sh[lane][0][q] = f0;
          C.sh[lane][1][q] = f1;
          s0 += f0;
          s1 += f1;
        }
        C.S[lane][0] = s0;
        C.S[lane][1] = s1;
      }
      __syncwarp();
      if (mfull | mplat) {
        // plateau events: V[q1][j] += 256 Sx[jx] Sy[jy] Sz[jz] for every
        // q1; lane (oi, oj) keeps component oj and the sum over j
        double vp = 0.0, gp = 0.0;
        for (unsigned mm = mplat; mm; mm &= mm - 1) {
          const int c = __ffs(mm) - 1;
          const int jx = (c < 8) ? (c & 1) : 2;
          const int jy = 3 + ((c < 8) ? ((c >> 1) & 1) : 2);
          const int jz = 6 + ((c < 8) ? ((c >> 2) & 1) : 2);
          vp = fma(C.S[jx][oj & 1] * C.S[jy][(oj >> 1) & 1],
                   C.S[jz][oj >> 2], vp);
          gp = fma((C.S[jx][0] + C.S[jx][1]) * (C.S[jy][0] + C.S[jy][1]),
                   C.S[jz][0] + C.S[jz][1], gp);
        }
        vp *= 256.0;
        gp *= 256.0;
        double b0 = s_pw[oi] * vp, b1 = s_pw[oi + 4] * vp;
        if (mfull) {
          double V[8];
#pragma unroll
          for (int j = 0; j < 8; j++) V[j] = 0.0;
          for (unsigned mm = mfull; mm; mm &= mm - 1) {
            const int c = __ffs(mm) - 1;
            const int ix = c & 1, iy = 3 + ((c >> 1) & 1),
                      iz = 6 + ((c >> 2) & 1);
            event_full2<NO>(P, C, ix, iy, iz, ys, V);
          }
          // b21[i][j] = -jac_in * sum_q1 phiw[q1][i] V[q1][j]
          if (active) {
#pragma unroll
            for (int j = 0; j < 8; j++) buf[lane][j] = V[j];
          }
#pragma unroll
          for (int j = 0; j < 8; j++) gp += V[j];
          __syncwarp();
#pragma unroll
          for (int q = 0; q < NQ1; q++) {
            const double v = buf[q][oj];
            const double2 pw = s_phiw2[q][oi];
            b0 = fma(pw.x, v, b0);
            b1 = fma(pw.y, v, b1);
          }
        }
        if (active) buf[lane][8] += gp;
        const double sc = -P.scale * C.jac_in;
        // both old values loaded before either store (distinct rows; the
        // compiler cannot prove it and would serialise the two RMWs)
        const double o0 = P.vals[slot0], o1 = P.vals[slot1];
        P.vals[slot0] = o0 + sc * b0;
        P.vals[slot1] = o1 + sc * b1;
      }
      __syncwarp();
    }
  }
  // A22 for the whole element: jac_in * sum_q1 G[q1] phiw[q1][i] phi[q1][j]
  __syncwarp();
  double b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int q = 0; q < NQ1; q++) {
    const double gq = buf[q][8] * s_phi[q][oj];
    const double2 pw = s_phiw2[q][oi];
    b0 = fma(pw.x, gq, b0);
    b1 = fma(pw.y, gq, b1);
  }
  const int64_t *mdofs = M.elem_dofs + m * M.nloc_max;
  const int64_t col = mdofs[oj];
  const double sc = P.scale * C.jac_in;
  P.vals[pat_index(P.pat, mdofs[oi], col)] += sc * b0;
  P.vals[pat_index(P.pat, mdofs[oi + 4], col)] += sc * b1;
  if (lane == 0) {
    unsigned long long *Cn = P.counters;
    counter_add(Cn + MF_CNT_EVENTS,
                (unsigned long long)cnt[1] + cnt[2] + cnt[3] + cnt[4]);
    counter_add(Cn + MF_CNT_PAIRS, cnt[0]);
    counter_add(Cn + MF_CNT_EV_UPPER, cnt[1]);
    counter_add(Cn + MF_CNT_EV_PLATEAU, cnt[2]);
    counter_add(Cn + MF_CNT_EV_DEAD, cnt[3]);
    counter_add(Cn + MF_CNT_EV_FULL, cnt[4]);
  }
}

template <int NO, int NI>
cudaError_t launch2(const AsmParams &P, cudaStream_t s) {
  const int64_t grid = (P.n_inner + kWarps2 - 1) / kWarps2;
  k_hex2<NO, NI><<<(unsigned)grid, kWarps2 * 32, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace

// L_max == 2 fast path of mf_hex_supported() meshes
bool mf_hex2_supported(const AsmParams &P) {
#ifdef MF_NO_HEX2  // A/B builds only
  return false;
#endif
  return P.L_max == 2 && P.shortcuts && P.eps > 0.0 &&
         !(P.flags & MF_FLAG_HEX_LEVELS);
}

cudaError_t mf_launch_hex2(const AsmParams &P, cudaStream_t s) {
  const int no = P.rules.n1d_box_out, ni = P.rules.n1d_box_in;
  if (ni == 3) {
    if (no == 2) return launch2<2, 3>(P, s);
    if (no == 3) return launch2<3, 3>(P, s);
    if (no == 4) return launch2<4, 3>(P, s);
  } else if (ni == 2) {
    if (no == 2) return launch2<2, 2>(P, s);
    if (no == 3) return launch2<3, 2>(P, s);
    if (no == 4) return launch2<4, 2>(P, s);
  }
  return cudaErrorNotSupported;
}
