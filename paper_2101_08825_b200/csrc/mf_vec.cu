// mf_vec.cu -- fused vector kernels of the device solver and host glue.
//
// Jacobi-preconditioned CG (solver.py:26-90) spends each iteration on one
// masked matvec and a handful of BLAS-1 updates and dot products.  They
// run here as three fused launches per iteration:
//   k_cg_matvec_dot  Ap = A p with constrained rows zeroed, and p.Ap
//   k_cg_update      x += a p; r -= a Ap; z = dinv r; and r.r, r.z
//   k_cg_direction   p = z + b p
// Reductions are deterministic: a fixed grid, a fixed per-block tree and a
// single-block pass over the block partials in block order (no atomics),
// so every run gives bit-identical iterates.  Also here: the indexed
// gather/scatter of assemble_rhs (rhs = load[free] - (A g)[free],
// assembly.py:691) and the ordered buffer sum / touched-row flags of the
// partitioned merge and ownership audit (parallel.py:180-200).
#include "mf_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 148 * 8;  // fixed: the reduction order depends on it

MF_DEV double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += sh[i];
  return s;  // valid in thread 0
}

struct RowBox {
  int xlo, ylo, zlo, Wx, Wy;
  int64_t p0;
};

MF_DEV RowBox row_box(const MfPattern &P, int64_t r) {
  RowBox b;
  const int rx = (int)(r % P.NX);
  const int64_t t = r / P.NX;
  const int ry = (int)(t % P.NY), rz = (int)(t / P.NY);
  b.xlo = max(rx - P.K, 0);
  b.ylo = max(ry - P.K, 0);
  b.zlo = max(rz - P.K, 0);
  b.Wx = min(rx + P.K, P.NX - 1) - b.xlo + 1;
  b.Wy = min(ry + P.K, P.NY - 1) - b.ylo + 1;
  b.p0 = P.rowptr[r];
  return b;
}

// Ap[r] = (cmask[r] ? 0 : sum_c A_rc p_c); partial[block] += p[r] Ap[r]
__global__ void __launch_bounds__(kThreads)
    k_cg_matvec_dot(MfPattern P, const double *vals, const double *p,
                    const uint8_t *cmask, double *Ap, double *partial) {
  __shared__ double sh[kThreads / 32];
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;  // lane 0 of each warp: its rows' p.Ap in row order
  for (int64_t r = w0; r < P.n; r += nw) {
    const RowBox b = row_box(P, r);
    const int ne = (int)(P.rowptr[r + 1] - b.p0);
    double s = 0.0;
    for (int e = lane; e < ne; e += 32) {
      const int ix = e % b.Wx, t = e / b.Wx;
      const int iy = t % b.Wy, iz = t / b.Wy;
      const int64_t c =
          ((int64_t)(b.zlo + iz) * P.NY + (b.ylo + iy)) * P.NX + (b.xlo + ix);
      s += vals[b.p0 + e] * p[c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (cmask[r]) s = 0.0;
    if (lane == 0) {
      Ap[r] = s;
      acc += p[r] * s;
    }
  }
  if (lane != 0) acc = 0.0;
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kThreads)
    k_cg_update(int64_t n, double alpha, const double *p, const double *Ap,
                const double *dinv, double *x, double *r, double *z,
                double *partial) {
  __shared__ double sh[kThreads / 32];
  double rr = 0.0, rz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    const double zi = dinv[i] * ri;
    z[i] = zi;
    rr += ri * ri;
    rz += ri * zi;
  }
  const double a = block_sum(rr, sh);
  const double b = block_sum(rz, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = a;
    partial[2 * blockIdx.x + 1] = b;
  }
}

// out[k] = sum over blocks of partial[block * stride + k], block order
__global__ void k_finish(const double *partial, int nblocks, int stride,
                         double *out) {
  const int k = threadIdx.x;
  if (k >= stride) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; b++) s += partial[b * stride + k];
  out[k] = s;
}

__global__ void k_cg_direction(int64_t n, double beta, const double *z,
                               double *p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// dinv = cmask ? 0 : 1/d; partial[block] = min over free rows of d
__global__ void __launch_bounds__(kThreads)
    k_jacobi(int64_t n, const double *d, const uint8_t *cmask, double *dinv,
             double *partial) {
  __shared__ double sh[kThreads / 32];
  double mn = INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool c = cmask[i];
    dinv[i] = c ? 0.0 : 1.0 / d[i];
    if (!c) mn = fmin(mn, d[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) m = fmin(m, sh[i]);
    partial[blockIdx.x] = m;
  }
}

__global__ void k_min_finish(const double *partial, int nblocks,
                             double *out) {
  double m = INFINITY;
  for (int b = 0; b < nblocks; b++) m = fmin(m, partial[b]);
  out[0] = m;
}

__global__ void k_gather_diff(int64_t n, const int64_t *idx, const double *a,
                              const double *b, double *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[k];
    out[k] = b ? a[i] - b[i] : a[i];
  }
}

__global__ void k_scatter(int64_t n, const int64_t *idx, const double *v,
                          double *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[idx[k]] = v[k];
}

struct BufList {
  const double *p[64];
};

__global__ void k_sum_ordered(BufList B, int nbuf, int64_t n, double scale,
                              double *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = B.p[0][i];
    for (int k = 1; k < nbuf; k++) s += B.p[k][i];
    out[i] = scale * s;
  }
}

// flags[r] = 1 if row r holds a nonzero value
__global__ void k_row_touched(MfPattern P, const double *vals,
                              uint8_t *flags) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < P.n; r += nw) {
    const int64_t a = P.rowptr[r], b = P.rowptr[r + 1];
    bool nz = false;
    for (int64_t e = a + lane; e < b; e += 32) nz |= vals[e] != 0.0;
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) flags[r] = nz;
  }
}

__global__ void k_axpby(int64_t n, double a, const double *x, double b,
                        const double *y, double *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

// y[r] = sum_c A_rc x_c for rows [row0, row1) (vals may be a window)
__global__ void k_matvec_rows(MfPattern P, const double *vals,
                              const double *x, int64_t row0, int64_t row1,
                              double *y) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = row0 + w0; r < row1; r += nw) {
    const RowBox b = row_box(P, r);
    const int ne = (int)(P.rowptr[r + 1] - b.p0);
    double s = 0.0;
    for (int e = lane; e < ne; e += 32) {
      const int ix = e % b.Wx, t = e / b.Wx;
      const int iy = t % b.Wy, iz = t / b.Wy;
      const int64_t c =
          ((int64_t)(b.zlo + iz) * P.NY + (b.ylo + iy)) * P.NX + (b.xlo + ix);
      s += vals[b.p0 + e] * x[c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = s;
  }
}

unsigned grid(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return (unsigned)(g < 148 * 32 ? (g > 0 ? g : 1) : 148 * 32);
}

}  // namespace

size_t mf_vec_ws_bytes() { return sizeof(double) * (2 * kBlocks + 64); }

cudaError_t mf_launch_cg_matvec_dot(const MfPattern &P, const double *vals,
                                    const double *p, const uint8_t *cmask,
                                    double *Ap, double *out, double *ws,
                                    cudaStream_t s) {
  k_cg_matvec_dot<<<kBlocks, kThreads, 0, s>>>(P, vals, p, cmask, Ap, ws);
  k_finish<<<1, 32, 0, s>>>(ws, kBlocks, 1, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_cg_update(int64_t n, double alpha, const double *p,
                                const double *Ap, const double *dinv,
                                double *x, double *r, double *z, double *out,
                                double *ws, cudaStream_t s) {
  k_cg_update<<<kBlocks, kThreads, 0, s>>>(n, alpha, p, Ap, dinv, x, r, z,
                                           ws);
  k_finish<<<1, 32, 0, s>>>(ws, kBlocks, 2, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_cg_direction(int64_t n, double beta, const double *z,
                                   double *p, cudaStream_t s) {
  if (n > 0) k_cg_direction<<<grid(n), kThreads, 0, s>>>(n, beta, z, p);
  return cudaGetLastError();
}

cudaError_t mf_launch_jacobi(int64_t n, const double *d, const uint8_t *cmask,
                             double *dinv, double *out_min, double *ws,
                             cudaStream_t s) {
  k_jacobi<<<kBlocks, kThreads, 0, s>>>(n, d, cmask, dinv, ws);
  k_min_finish<<<1, 1, 0, s>>>(ws, kBlocks, out_min);
  return cudaGetLastError();
}

cudaError_t mf_launch_gather_diff(int64_t n, const int64_t *idx,
                                  const double *a, const double *b,
                                  double *out, cudaStream_t s) {
  if (n > 0) k_gather_diff<<<grid(n), kThreads, 0, s>>>(n, idx, a, b, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_scatter(int64_t n, const int64_t *idx, const double *v,
                              double *out, cudaStream_t s) {
  if (n > 0) k_scatter<<<grid(n), kThreads, 0, s>>>(n, idx, v, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_sum_ordered(int nbuf, const double *const *bufs,
                                  int64_t n, double scale, double *out,
                                  cudaStream_t s) {
  BufList B;
  for (int k = 0; k < nbuf; k++) B.p[k] = bufs[k];
  if (n > 0) k_sum_ordered<<<grid(n), kThreads, 0, s>>>(B, nbuf, n, scale, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_row_touched(const MfPattern &P, const double *vals,
                                  uint8_t *flags, cudaStream_t s) {
  if (P.n > 0) {
    const int64_t want = (P.n * 32 + kThreads - 1) / kThreads;
    const unsigned g = (unsigned)(want < 148 * 32 ? want : 148 * 32);
    k_row_touched<<<g, kThreads, 0, s>>>(P, vals, flags);
  }
  return cudaGetLastError();
}

cudaError_t mf_launch_axpby(int64_t n, double a, const double *x, double b,
                            const double *y, double *out, cudaStream_t s) {
  if (n > 0) k_axpby<<<grid(n), kThreads, 0, s>>>(n, a, x, b, y, out);
  return cudaGetLastError();
}

cudaError_t mf_launch_matvec_rows(const MfPattern &P, const double *vals,
                                  const double *x, int64_t row0, int64_t row1,
                                  double *y, cudaStream_t s) {
  if (row1 > row0) {
    const int64_t want = ((row1 - row0) * 32 + kThreads - 1) / kThreads;
    const unsigned g = (unsigned)(want < 148 * 32 ? want : 148 * 32);
    k_matvec_rows<<<g, kThreads, 0, s>>>(P, vals, x, row0, row1, y);
  }
  return cudaGetLastError();
}
