// mf_lists.cu -- explicit candidate lists for mf_general_core_lists.
//
// _general_core (_kernels.py:391-487) takes its pairs as CSR lists per
// OUTER element (outer_ids, cand_ptr, cand_ids).  All of a pair's blocks
// land in rows of its INNER element (_kernels.py:483-486), so the device
// path wants them per inner element: the lists are transposed here with a
// stable radix sort on the inner id (pairs of one inner element keep the
// caller's order), run-length encoded into per-element ranges, and each
// pair's outer id is looked up by binary search in cand_ptr.
#include <cub/cub.cuh>

#include "mf_lists.cuh"

namespace {

__global__ void k_iota(int64_t *v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

// list_outer[k] = outer_ids[i] with cand_ptr[i] <= pidx[k] < cand_ptr[i+1]
__global__ void k_list_outer(const int64_t *cand_ptr, int64_t n_outer,
                             const int64_t *outer_ids, const int64_t *pidx,
                             int64_t npairs, int64_t *list_outer) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       k < npairs; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pidx[k];
    int64_t lo = 0, hi = n_outer;  // invariant: cand_ptr[lo] <= p
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (cand_ptr[mid] <= p)
        lo = mid;
      else
        hi = mid;
    }
    list_outer[k] = outer_ids[lo];
  }
}

__global__ void k_gather_dofs(const int64_t *elem_dofs, int nloc,
                              const int64_t *uniq, int64_t n,
                              int64_t *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       i < n * nloc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / nloc;
    out[i] = elem_dofs[uniq[t] * nloc + (i - t * nloc)];
  }
}

unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

int bits_for(int64_t n) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) < n) b++;
  return b;
}

}  // namespace

#define MF_TRY(x)                          \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)

cudaError_t mf_lists_build(const int64_t *cand_ptr, const int64_t *cand_ids,
                           const int64_t *outer_ids, int64_t n_outer,
                           int64_t npairs, int64_t n_elem,
                           const int64_t *elem_dofs, int nloc,
                           cudaStream_t s, MfLists &L) {
  L = MfLists();
  L.npairs = npairs;
  MF_TRY(cudaMallocAsync(&L.pidx_in, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.keys, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.pidx, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.list_outer, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.uniq, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.counts, 8 * npairs, s));
  MF_TRY(cudaMallocAsync(&L.nruns, 8, s));
  k_iota<<<grid_for(npairs), 256, 0, s>>>(L.pidx_in, npairs);
  MF_TRY(cudaGetLastError());
  const int bits = bits_for(n_elem);
  size_t b1 = 0, b2 = 0;
  MF_TRY(cub::DeviceRadixSort::SortPairs(
      nullptr, b1, cand_ids, L.keys, L.pidx_in, L.pidx, npairs, 0, bits, s));
  MF_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, b2, L.keys, L.uniq,
                                            L.counts, L.nruns, npairs, s));
  L.tmp_bytes = b1 > b2 ? b1 : b2;
  MF_TRY(cudaMallocAsync(&L.tmp, L.tmp_bytes, s));
  // stable: pairs of one inner element stay in the caller's list order
  MF_TRY(cub::DeviceRadixSort::SortPairs(L.tmp, L.tmp_bytes, cand_ids,
                                         L.keys, L.pidx_in, L.pidx, npairs, 0,
                                         bits, s));
  MF_TRY(cub::DeviceRunLengthEncode::Encode(L.tmp, L.tmp_bytes, L.keys,
                                            L.uniq, L.counts, L.nruns, npairs,
                                            s));
  k_list_outer<<<grid_for(npairs), 256, 0, s>>>(cand_ptr, n_outer, outer_ids,
                                                 L.pidx, npairs,
                                                 L.list_outer);
  MF_TRY(cudaGetLastError());
  MF_TRY(cudaMemcpyAsync(&L.n_inner, L.nruns, 8, cudaMemcpyDeviceToHost, s));
  MF_TRY(cudaStreamSynchronize(s));
  const int64_t n = L.n_inner;
  L.h_uniq.resize(n);
  L.h_counts.resize(n);
  L.h_dofs.resize(n * nloc);
  MF_TRY(cudaMemcpyAsync(L.h_uniq.data(), L.uniq, 8 * n,
                         cudaMemcpyDeviceToHost, s));
  MF_TRY(cudaMemcpyAsync(L.h_counts.data(), L.counts, 8 * n,
                         cudaMemcpyDeviceToHost, s));
  MF_TRY(cudaStreamSynchronize(s));
  // every inner id in range before the device gather reads elem_dofs
  for (int64_t i = 0; i < n; i++)
    if (L.h_uniq[i] < 0 || L.h_uniq[i] >= n_elem) return cudaErrorInvalidValue;
  int64_t *gd = nullptr;
  MF_TRY(cudaMallocAsync(&gd, 8 * (n * nloc > 0 ? n * nloc : 1), s));
  k_gather_dofs<<<grid_for(n * nloc), 256, 0, s>>>(elem_dofs, nloc, L.uniq, n,
                                                    gd);
  MF_TRY(cudaGetLastError());
  MF_TRY(cudaMemcpyAsync(L.h_dofs.data(), gd, 8 * n * nloc,
                         cudaMemcpyDeviceToHost, s));
  MF_TRY(cudaStreamSynchronize(s));
  MF_TRY(cudaFreeAsync(gd, s));
  return cudaSuccess;
}

void mf_lists_free(MfLists &L, cudaStream_t s) {
  void *p[] = {L.pidx_in, L.keys, L.pidx, L.list_outer, L.uniq,
               L.counts,  L.nruns, L.tmp};
  for (void *q : p)
    if (q) cudaFreeAsync(q, s);
  L = MfLists();
}
