// mf_candidates.cu -- element-pair neighbour search on the cell grid.
//
// Replaces _count_candidates / _fill_candidates (_kernels.py:1205-1268) and
// the host cumsum between them (assembly.py:157-175).  One warp per outer
// element: the lanes take 32 consecutive cells of the clipped (2R+1)^dim
// stencil in lex order (z, y, x) -- the reference's loop order -- test every
// element of their cell with the reference's max-axis gap (< reach,
// strict), and a warp prefix sum over the per-lane hit counts places the
// ids.  Cells are visited in ascending order and elements are cell-lex
// ordered, so ids come out ascending exactly like the reference.
#include <cub/device/device_scan.cuh>

#include "mf_common.cuh"

namespace {

template <int DIM, bool FILL>
__global__ void __launch_bounds__(256)
    k_candidates(MfMesh M, const int64_t *outer_ids, int64_t n_outer,
                 const uint8_t *inner_mask, int R, double reach,
                 int64_t *counts, const int64_t *ptr, int64_t *ids) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t oi = warp; oi < n_outer; oi += nwarps) {
    const int64_t l = outer_ids[oi];
    int cx, cy, cz;
    cell_coords(M.elem_cell[l], M.ncx, M.ncy, cx, cy, cz);
    const int xlo = max(cx - R, 0), xhi = min(cx + R, M.ncx - 1);
    const int ylo = max(cy - R, 0), yhi = min(cy + R, M.ncy - 1);
    const int zlo = DIM == 3 ? max(cz - R, 0) : 0;
    const int zhi = DIM == 3 ? min(cz + R, M.ncz - 1) : 0;
    const int nx = xhi - xlo + 1, ny = yhi - ylo + 1, nz = zhi - zlo + 1;
    const int ncell = nx * ny * nz;
    double llo[DIM], lhi[DIM];
#pragma unroll
    for (int k = 0; k < DIM; k++) {
      llo[k] = M.elem_lo[l * DIM + k];
      lhi[k] = M.elem_hi[l * DIM + k];
    }
    int64_t p = FILL ? ptr[oi] : 0;
    for (int base = 0; base < ncell; base += 32) {
      const int i = base + lane;
      int hits = 0;
      int64_t e0 = 0, e1 = 0;
      if (i < ncell) {
        const int x2 = xlo + i % nx;
        const int t = i / nx;
        const int y2 = ylo + t % ny;
        const int z2 = zlo + t / ny;
        const int64_t c2 = ((int64_t)z2 * M.ncy + y2) * M.ncx + x2;
        e0 = M.cell_ptr[c2];
        e1 = M.cell_ptr[c2 + 1];
        for (int64_t e = e0; e < e1; e++) {
          if (!inner_mask[e]) continue;
          double gap = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; k++) {
            double d1 = xsub(llo[k], M.elem_hi[e * DIM + k]);
            double d2 = xsub(M.elem_lo[e * DIM + k], lhi[k]);
            if (d1 > gap) gap = d1;
            if (d2 > gap) gap = d2;
          }
          if (gap < reach) hits++;
        }
      }
      // inclusive warp scan of hits
      int incl = hits;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (FILL && hits) {
        int64_t q = p + incl - hits;
        for (int64_t e = e0; e < e1; e++) {
          if (!inner_mask[e]) continue;
          double gap = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; k++) {
            double d1 = xsub(llo[k], M.elem_hi[e * DIM + k]);
            double d2 = xsub(M.elem_lo[e * DIM + k], lhi[k]);
            if (d1 > gap) gap = d1;
            if (d2 > gap) gap = d2;
          }
          if (gap < reach) ids[q++] = e;
        }
      }
      p += total;
    }
    if (!FILL && lane == 0) counts[oi] = p;
  }
}

}  // namespace

cudaError_t mf_launch_candidates(const MfMesh &M, const int64_t *outer_ids,
                                 int64_t n_outer, const uint8_t *inner_mask,
                                 int R, double reach, int64_t *counts,
                                 const int64_t *ptr, int64_t *ids,
                                 cudaStream_t s) {
  if (n_outer <= 0) return cudaSuccess;
  const int block = 256;
  int64_t want = (n_outer * 32 + block - 1) / block;
  int grid = (int)(want < 148 * 64 ? want : 148 * 64);
  bool fill = ids != nullptr;
  if (M.dim == 2) {
    if (fill)
      k_candidates<2, true><<<grid, block, 0, s>>>(M, outer_ids, n_outer,
                                                   inner_mask, R, reach,
                                                   counts, ptr, ids);
    else
      k_candidates<2, false><<<grid, block, 0, s>>>(M, outer_ids, n_outer,
                                                    inner_mask, R, reach,
                                                    counts, ptr, ids);
  } else {
    if (fill)
      k_candidates<3, true><<<grid, block, 0, s>>>(M, outer_ids, n_outer,
                                                   inner_mask, R, reach,
                                                   counts, ptr, ids);
    else
      k_candidates<3, false><<<grid, block, 0, s>>>(M, outer_ids, n_outer,
                                                    inner_mask, R, reach,
                                                    counts, ptr, ids);
  }
  return cudaGetLastError();
}

namespace {
__global__ void k_zero_first(int64_t *ptr) { ptr[0] = 0; }
}  // namespace

size_t mf_scan_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t *)nullptr,
                                (int64_t *)nullptr, (int)(n > 0 ? n : 1));
  return bytes;
}

cudaError_t mf_scan(const int64_t *counts, int64_t n, int64_t *ptr, void *ws,
                    size_t ws_bytes, cudaStream_t s) {
  k_zero_first<<<1, 1, 0, s>>>(ptr);
  if (n <= 0) return cudaGetLastError();
  return cub::DeviceScan::InclusiveSum(ws, ws_bytes, counts, ptr + 1, (int)n,
                                       s);
}
