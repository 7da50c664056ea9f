// mf_lists.cuh -- device transposition of explicit candidate lists
// (mf_lists.cu), used by mf_general_core_lists (mf_capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

struct MfLists {
  // device, npairs entries each: pair index order, sorted inner ids,
  // pair positions (stable), outer id per sorted pair
  int64_t *pidx_in = nullptr, *keys = nullptr, *pidx = nullptr;
  int64_t *list_outer = nullptr;
  // device run-length encoding of the sorted inner ids
  int64_t *uniq = nullptr, *counts = nullptr, *nruns = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int64_t npairs = 0, n_inner = 0;
  // host copies: distinct inner elements (ascending), their pair counts
  // and DOF rows (n_inner x nloc) for the colouring
  std::vector<int64_t> h_uniq, h_counts, h_dofs;
};

cudaError_t mf_lists_build(const int64_t *cand_ptr, const int64_t *cand_ids,
                           const int64_t *outer_ids, int64_t n_outer,
                           int64_t npairs, int64_t n_elem,
                           const int64_t *elem_dofs, int nloc,
                           cudaStream_t s, MfLists &L);
void mf_lists_free(MfLists &L, cudaStream_t s);
