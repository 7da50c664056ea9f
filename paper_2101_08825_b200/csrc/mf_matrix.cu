// mf_matrix.cu -- operations on the implicit structured pattern.
//
// Device versions of the reference's matrix utilities (_kernels.py:846-1202)
// used by _finish (assembly.py:440-445), the solver (solver.py:42-52) and
// assemble_rhs (assembly.py:691).  One warp per row: the row's entries are
// the clipped (2K+1)^dim grid box around the row, stored x-fastest, so a
// warp walks them with coalesced loads.  Reductions that produce a max use
// an integer atomicMax on the (non-negative) double bit pattern, which is
// order independent and therefore deterministic.
#include "mf_common.cuh"

namespace {

struct RowBox {
  int xlo, xhi, ylo, yhi, zlo, zhi, Wx, Wy;
  int64_t p0;
};

MF_DEV RowBox row_box(const MfPattern &P, int64_t r) {
  RowBox b;
  int rx = (int)(r % P.NX);
  int64_t t = r / P.NX;
  int ry = (int)(t % P.NY), rz = (int)(t / P.NY);
  b.xlo = max(rx - P.K, 0);
  b.xhi = min(rx + P.K, P.NX - 1);
  b.ylo = max(ry - P.K, 0);
  b.yhi = min(ry + P.K, P.NY - 1);
  b.zlo = max(rz - P.K, 0);
  b.zhi = min(rz + P.K, P.NZ - 1);
  b.Wx = b.xhi - b.xlo + 1;
  b.Wy = b.yhi - b.ylo + 1;
  b.p0 = P.rowptr[r];
  return b;
}

// column of the e-th entry of a row
MF_DEV int64_t entry_col(const MfPattern &P, const RowBox &b, int e) {
  int ix = e % b.Wx;
  int t = e / b.Wx;
  int iy = t % b.Wy;
  int iz = t / b.Wy;
  return ((int64_t)(b.zlo + iz) * P.NY + (b.ylo + iy)) * P.NX + (b.xlo + ix);
}

MF_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

MF_DEV void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr),
            (unsigned long long)__double_as_longlong(v));
}

#define WARP_ROWS_BEGIN                                                   \
  const int lane = threadIdx.x & 31;                                      \
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; \
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;              \
  for (int64_t r = w0; r < P.n; r += nw) {                                \
    const RowBox b = row_box(P, r);                                       \
    const int ne = (int)(P.rowptr[r + 1] - b.p0);

__global__ void k_asym(MfPattern P, const double *vals, double *out) {
  WARP_ROWS_BEGIN
  double s = 0.0;
  for (int e = lane; e < ne; e += 32) {
    int64_t c = entry_col(P, b, e);
    s += fabs(vals[b.p0 + e] - vals[pat_index(P, c, r)]);
  }
  s = warp_sum(s);
  if (lane == 0) atomic_max_nonneg(out, s);
}
}

// rows [row0, row1) only (distributed row blocks: vals may be a window
// holding the rows within K planes of the range)
__global__ void k_asym_rows(MfPattern P, const double *vals, int64_t row0,
                            int64_t row1, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = row0 + w0; r < row1; r += nw) {
    const RowBox b = row_box(P, r);
    const int ne = (int)(P.rowptr[r + 1] - b.p0);
    double s = 0.0;
    for (int e = lane; e < ne; e += 32) {
      int64_t c = entry_col(P, b, e);
      s += fabs(vals[b.p0 + e] - vals[pat_index(P, c, r)]);
    }
    s = warp_sum(s);
    if (lane == 0) atomic_max_nonneg(out, s);
  }
}

__global__ void k_norm(MfPattern P, const double *vals, double *out) {
  WARP_ROWS_BEGIN
  double s = 0.0;
  for (int e = lane; e < ne; e += 32) s += fabs(vals[b.p0 + e]);
  s = warp_sum(s);
  if (lane == 0) atomic_max_nonneg(out, s);
}
}

__global__ void k_matvec(MfPattern P, const double *vals, const double *x,
                         double *y) {
  WARP_ROWS_BEGIN
  double s = 0.0;
  for (int e = lane; e < ne; e += 32)
    s += vals[b.p0 + e] * x[entry_col(P, b, e)];
  s = warp_sum(s);
  if (lane == 0) y[r] = s;
}
}

__global__ void k_symmetrize(MfPattern P, double *vals) {
  WARP_ROWS_BEGIN
  for (int e = lane; e < ne; e += 32) {
    int64_t c = entry_col(P, b, e);
    if (c > r) {
      int64_t q = pat_index(P, c, r);
      double a = 0.5 * (vals[b.p0 + e] + vals[q]);
      vals[b.p0 + e] = a;
      vals[q] = a;
    }
  }
}
}

__global__ void k_fill_cols(MfPattern P, int64_t *cols) {
  WARP_ROWS_BEGIN
  for (int e = lane; e < ne; e += 32) cols[b.p0 + e] = entry_col(P, b, e);
}
}

__global__ void k_diag(MfPattern P, const double *vals, double *out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < P.n) out[r] = vals[pat_index(P, r, r)];
}

__global__ void k_scale(double *v, int64_t n, double s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) v[i] *= s;
}

__global__ void k_probe(double *out, int64_t iters) {
  // 8 independent DFMA chains per thread
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9,
         a3 = a0 + 3e-9, a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9,
         a7 = a0 + 7e-9;
  const double b = 0.999999999, c = 1e-12;
  for (int64_t i = 0; i < iters; i++) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c);
    a3 = fma(a3, b, c); a4 = fma(a4, b, c); a5 = fma(a5, b, c);
    a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// one thread per element of a colour: contract f*w*|J| with the shapes and
// add into the element's DOFs (race-free inside a colour)
__global__ void k_load(MfMesh M, const int32_t *elems, int64_t n,
                       const double *fval, const double *w, const double *phi,
                       int nq, int nloc, double *load) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t e = elems[k];
  const int dim = M.dim;
  double det;
  if (M.elem_kind[e] == 3) {  // tetrahedron: |det| of the edge matrix
    const double *c = M.elem_coords + e * M.nv_max * 3;
    double a[3], b[3], d[3];
    for (int k = 0; k < 3; k++) {
      a[k] = c[3 + k] - c[k];
      b[k] = c[6 + k] - c[k];
      d[k] = c[9 + k] - c[k];
    }
    det = fabs(a[0] * (b[1] * d[2] - b[2] * d[1]) +
               a[1] * (b[2] * d[0] - b[0] * d[2]) +
               a[2] * (b[0] * d[1] - b[1] * d[0]));
  } else if (M.elem_kind[e] == 1) {
    const double *c = M.elem_coords + e * M.nv_max * dim;
    const double e10 = c[dim] - c[0], e11 = c[dim + 1] - c[1];
    const double e20 = c[2 * dim] - c[0], e21 = c[2 * dim + 1] - c[1];
    det = e10 * e21 - e11 * e20;
  } else {
    det = 1.0;
    for (int a = 0; a < dim; a++)
      det *= 0.5 * (M.elem_hi[e * dim + a] - M.elem_lo[e * dim + a]);
  }
  const double *fv = fval + k * nq;
  for (int i = 0; i < nloc; i++) {
    double s = 0.0;
    for (int q = 0; q < nq; q++) s += fv[q] * w[q] * phi[q * nloc + i];
    load[M.elem_dofs[e * M.nloc_max + i]] += det * s;
  }
}

int rows_grid(int64_t n) {
  int64_t want = (n * 32 + 255) / 256;
  return (int)(want < 148 * 32 ? (want > 0 ? want : 1) : 148 * 32);
}

}  // namespace

cudaError_t mf_launch_asym(const MfPattern &P, const double *vals,
                           double *out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  k_asym<<<rows_grid(P.n), 256, 0, s>>>(P, vals, out);
  return cudaGetLastError();
}
cudaError_t mf_launch_asym_rows(const MfPattern &P, const double *vals,
                                int64_t row0, int64_t row1, double *out,
                                cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  if (row1 > row0)
    k_asym_rows<<<rows_grid(row1 - row0), 256, 0, s>>>(P, vals, row0, row1,
                                                         out);
  return cudaGetLastError();
}
cudaError_t mf_launch_norm(const MfPattern &P, const double *vals,
                           double *out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
  if (e != cudaSuccess) return e;
  k_norm<<<rows_grid(P.n), 256, 0, s>>>(P, vals, out);
  return cudaGetLastError();
}
cudaError_t mf_launch_matvec(const MfPattern &P, const double *vals,
                             const double *x, double *y, cudaStream_t s) {
  k_matvec<<<rows_grid(P.n), 256, 0, s>>>(P, vals, x, y);
  return cudaGetLastError();
}
cudaError_t mf_launch_symmetrize(const MfPattern &P, double *vals,
                                 cudaStream_t s) {
  k_symmetrize<<<rows_grid(P.n), 256, 0, s>>>(P, vals);
  return cudaGetLastError();
}
cudaError_t mf_launch_fill_cols(const MfPattern &P, int64_t *cols,
                                cudaStream_t s) {
  k_fill_cols<<<rows_grid(P.n), 256, 0, s>>>(P, cols);
  return cudaGetLastError();
}
cudaError_t mf_launch_diag(const MfPattern &P, const double *vals,
                           double *out, cudaStream_t s) {
  if (P.n > 0) k_diag<<<(int)((P.n + 255) / 256), 256, 0, s>>>(P, vals, out);
  return cudaGetLastError();
}
cudaError_t mf_launch_scale(double *v, int64_t n, double sc, cudaStream_t s) {
  if (n > 0) {
    int64_t want = (n + 255) / 256;
    k_scale<<<(int)(want < 148 * 64 ? want : 148 * 64), 256, 0, s>>>(v, n,
                                                                     sc);
  }
  return cudaGetLastError();
}
cudaError_t mf_launch_load(const MfMesh &M, const int32_t *elems, int64_t n,
                           const double *fval, const double *w,
                           const double *phi, int nq, int nloc, double *load,
                           cudaStream_t s) {
  if (n > 0)
    k_load<<<(int)((n + 127) / 128), 128, 0, s>>>(M, elems, n, fval, w, phi,
                                                   nq, nloc, load);
  return cudaGetLastError();
}
cudaError_t mf_launch_probe(double *out, int64_t iters, int blocks,
                            int threads, cudaStream_t s) {
  k_probe<<<blocks, threads, 0, s>>>(out, iters);
  return cudaGetLastError();
}
