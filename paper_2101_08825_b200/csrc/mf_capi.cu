// mf_capi.cu -- extern "C" entry points of include/mollifem_b200.h.
//
// Argument validation, launch configuration and kernel selection live
// here; the kernels are in mf_candidates.cu, mf_generic.cu, mf_hex.cu,
// mf_2d.cu and mf_matrix.cu.  Host arithmetic that feeds classification
// (delta -/+ eps and their squares, _kernels.py:410-413) is plain IEEE
// double without contraction (x86-64 host code, no -mfma).
#include <cstring>
#include <string>

#include <algorithm>

#include <vector>

#include "mf_common.cuh"
#include "mf_lists.cuh"

cudaError_t mf_launch_candidates(const MfMesh &, const int64_t *, int64_t,
                                 const uint8_t *, int, double, int64_t *,
                                 const int64_t *, int64_t *, cudaStream_t);
size_t mf_scan_bytes(int64_t n);
cudaError_t mf_scan(const int64_t *, int64_t, int64_t *, void *, size_t,
                    cudaStream_t);
cudaError_t mf_launch_generic(const AsmParams &, int, int, cudaStream_t);
cudaError_t mf_launch_blocks(const AsmParams &, int, int, int, double,
                             const double *, double *, double *,
                             unsigned long long *, int64_t, cudaStream_t);
cudaError_t mf_launch_blocked_a22(const AsmParams &, int, int, int,
                                  const double *, const double *,
                                  const unsigned long long *, double *,
                                  double *, cudaStream_t);
cudaError_t mf_launch_blocked_gather(const AsmParams &, int, int, int,
                                     const double *, const double *, int64_t,
                                     int64_t, cudaStream_t);
int64_t mf_gather_table_doubles(int, int, int);
cudaError_t mf_launch_blocked_scatter(const AsmParams &, int, int, int,
                                      const int32_t *, const int64_t *,
                                      const double *, const double *,
                                      const unsigned long long *,
                                      cudaStream_t);
// specialised kernels: return cudaErrorNotSupported when they do not cover
// the configuration
cudaError_t mf_launch_hex(const AsmParams &, cudaStream_t);
cudaError_t mf_launch_2d(const AsmParams &, cudaStream_t);
bool mf_hex_supported(const AsmParams &);
cudaError_t mf_launch_hex2(const AsmParams &, cudaStream_t);
bool mf_hex2_supported(const AsmParams &);
bool mf_2d_supported(const AsmParams &);
cudaError_t mf_launch_tet(const AsmParams &, double *, cudaStream_t);
size_t mf_tet_scratch_doubles(const AsmParams &, int64_t);
bool mf_tet_supported(const AsmParams &);
cudaError_t mf_launch_tri_u(const AsmParams &, double *, cudaStream_t);
size_t mf_tri_u_scratch_doubles(const AsmParams &, int64_t);
bool mf_tri_u_supported(const AsmParams &);
cudaError_t mf_launch_asym(const MfPattern &, const double *, double *,
                           cudaStream_t);
cudaError_t mf_launch_norm(const MfPattern &, const double *, double *,
                           cudaStream_t);
cudaError_t mf_launch_asym_rows(const MfPattern &, const double *, int64_t,
                                int64_t, double *, cudaStream_t);
cudaError_t mf_launch_matvec(const MfPattern &, const double *,
                             const double *, double *, cudaStream_t);
cudaError_t mf_launch_symmetrize(const MfPattern &, double *, cudaStream_t);
cudaError_t mf_launch_fill_cols(const MfPattern &, int64_t *, cudaStream_t);
cudaError_t mf_launch_diag(const MfPattern &, const double *, double *,
                           cudaStream_t);
cudaError_t mf_launch_scale(double *, int64_t, double, cudaStream_t);
cudaError_t mf_launch_probe(double *, int64_t, int, int, cudaStream_t);
size_t mf_vec_ws_bytes();
cudaError_t mf_launch_cg_matvec_dot(const MfPattern &, const double *,
                                    const double *, const uint8_t *, double *,
                                    double *, double *, cudaStream_t);
cudaError_t mf_launch_cg_update(int64_t, double, const double *,
                                const double *, const double *, double *,
                                double *, double *, double *, double *,
                                cudaStream_t);
cudaError_t mf_launch_cg_direction(int64_t, double, const double *, double *,
                                   cudaStream_t);
cudaError_t mf_launch_jacobi(int64_t, const double *, const uint8_t *,
                             double *, double *, double *, cudaStream_t);
cudaError_t mf_launch_gather_diff(int64_t, const int64_t *, const double *,
                                  const double *, double *, cudaStream_t);
cudaError_t mf_launch_scatter(int64_t, const int64_t *, const double *,
                              double *, cudaStream_t);
cudaError_t mf_launch_sum_ordered(int, const double *const *, int64_t, double,
                                  double *, cudaStream_t);
cudaError_t mf_launch_row_touched(const MfPattern &, const double *,
                                  uint8_t *, cudaStream_t);
cudaError_t mf_launch_axpby(int64_t, double, const double *, double,
                            const double *, double *, cudaStream_t);
cudaError_t mf_launch_matvec_rows(const MfPattern &, const double *,
                                  const double *, int64_t, int64_t, double *,
                                  cudaStream_t);
cudaError_t mf_launch_load(const MfMesh &, const int32_t *, int64_t,
                           const double *, const double *, const double *,
                           int, int, double *, cudaStream_t);

#ifndef MF_SMALL_TRI_ELEMS
#define MF_SMALL_TRI_ELEMS 65536
#endif
#ifndef MF_KEEP_POOL
#define MF_KEEP_POOL 1
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

int cuda_status(cudaError_t e, const char *where) {
  if (e == cudaSuccess) return MF_OK;
  return fail(MF_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Reject host pointers early: a kernel handed a host address would fault
// asynchronously with "illegal memory access" far from the cause.
int check_dev(const void *p, const char *name) {
  if (!p) return MF_OK;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return fail(MF_ERR_ARG, std::string(name) + " is not a CUDA pointer");
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(MF_ERR_ARG, std::string(name) + " is not device memory");
  return MF_OK;
}

#define MF_CHECK_DEV(p)                          \
  do {                                           \
    if (int rc_ = check_dev((p), #p)) return rc_; \
  } while (0)

int check_mesh(const MfMesh *m) {
  if (!m) return fail(MF_ERR_ARG, "mesh is NULL");
  if (m->dim != 2 && m->dim != 3) return fail(MF_ERR_ARG, "dim must be 2/3");
  if (m->degree != 1 && m->degree != 2)
    return fail(MF_ERR_ARG, "degree must be 1/2");
  if (m->n_elem < 0) return fail(MF_ERR_ARG, "n_elem < 0");
  if (m->n_elem > 0 && (!m->elem_kind || !m->elem_lo || !m->elem_hi ||
                        !m->elem_cell || !m->cell_ptr))
    return fail(MF_ERR_ARG, "mesh array is NULL");
  if (m->ncx < 1 || m->ncy < 1 || m->ncz < 1)
    return fail(MF_ERR_ARG, "bad cell grid");
  if (int rc = check_dev(m->elem_lo, "mesh.elem_lo")) return rc;
  if (int rc = check_dev(m->elem_dofs, "mesh.elem_dofs")) return rc;
  return MF_OK;
}

int check_pattern(const MfPattern *p) {
  if (!p) return fail(MF_ERR_ARG, "pattern is NULL");
  if (p->n > 0 && !p->rowptr) return fail(MF_ERR_ARG, "rowptr is NULL");
  if (int rc = check_dev(p->rowptr, "pattern.rowptr")) return rc;
  if (p->NX < 1 || p->NY < 1 || p->NZ < 1 || p->K < 0)
    return fail(MF_ERR_ARG, "bad pattern grid");
  if ((int64_t)p->NX * p->NY * p->NZ != p->n)
    return fail(MF_ERR_ARG, "pattern grid does not match n");
  return MF_OK;
}

// keep freed call-scoped scratch (cudaMallocAsync / cudaFreeAsync) in the
// device's default pool across calls: release threshold 0 would unmap and
// remap it at every synchronisation.  Per-device setting, idempotent.
void keep_pool() {
#if MF_KEEP_POOL
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
#endif
}

constexpr int kGenericBlock = 128;
constexpr int kGenericMaxGrid = 148 * 4;

int nq_in_max(const MfRules *r) {
  return r->nq_box_in > r->nq_tri_in ? r->nq_box_in : r->nq_tri_in;
}

AsmParams make_params(const MfMesh *mesh, const MfRules *rules,
                      const MfKernel *kern, const MfPattern *pat,
                      const uint8_t *outer_mask, int32_t R, double scale,
                      double *vals, uint64_t *counters, int32_t flags) {
  AsmParams P;
  memset(&P, 0, sizeof(P));
  P.mesh = *mesh;
  P.rules = *rules;
  if (pat) P.pat = *pat;
  P.outer_mask = outer_mask;
  P.R = R;
  P.scale = scale;
  P.vals = vals;
  P.counters = reinterpret_cast<unsigned long long *>(counters);
  P.flags = flags;
  P.L_min = kern->L_min;
  P.L_max = kern->L_max;
  P.delta = kern->delta;
  P.eps = kern->eps;
  P.cde = kern->cde;
  const double dm = kern->delta - kern->eps;
  const double dp = kern->delta + kern->eps;
  P.dme = dm;
  P.dpe = dp;
  P.dm2 = dm * dm;
  P.dp2 = dp * dp;
  P.dme2_lo = dm * dm * (1.0 - 4e-12);
  P.dme2_hi = dm * dm * (1.0 + 4e-12);
  P.inv_eps = kern->eps > 0.0 ? 1.0 / kern->eps : 0.0;
  P.alpha = kern->delta * P.inv_eps;
  P.alpha2 = 2.0 * P.alpha;
  P.half_inv_eps = 0.5 * P.inv_eps;
  {
    int64_t b;
    memcpy(&b, &P.dm2, 8);
    P.hi_dm2 = (int32_t)(b >> 32);
    memcpy(&b, &P.dp2, 8);
    P.hi_dp2 = (int32_t)(b >> 32);
    P.hd_lo = P.hi_dm2 - 1;
    P.hd_hi = P.hi_dp2 + 1;
    // scaled shell edges: r = alpha - sqrt(q) leaves [-1, 1] by at most
    // 2^-20 relative there, where xi is flat to fourth order
    double ql = (P.alpha - 1.0) * (P.alpha - 1.0);
    double qh = (P.alpha + 1.0) * (P.alpha + 1.0);
    memcpy(&b, &ql, 8);
    P.hq_lo = (int32_t)(b >> 32) - 1;
    memcpy(&b, &qh, 8);
    P.hq_hi = (int32_t)(b >> 32) + 1;
  }
  P.nl_box = mesh->dim == 3 ? (mesh->degree + 1) * (mesh->degree + 1) *
                                  (mesh->degree + 1)
                            : (mesh->degree + 1) * (mesh->degree + 1);
  // simplex slots: triangles (3 * degree) in 2D, P1 tetrahedra in 3D
  P.nl_tri = mesh->dim == 3 ? 4 : 3 * mesh->degree;
  P.shortcuts = (flags & MF_FLAG_NO_SHORTCUTS) == 0 && kern->eps > 0.0;
  return P;
}

}  // namespace

extern "C" {

const char *mf_last_error(void) { return g_err.c_str(); }
int mf_abi_version(void) { return MF_ABI_VERSION; }

int mf_count_candidates(const MfMesh *mesh, const int64_t *outer_ids,
                        int64_t n_outer, const uint8_t *inner_mask,
                        int32_t R, double reach, int64_t *counts,
                        void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (n_outer < 0 || R < 1) return fail(MF_ERR_ARG, "bad n_outer/R");
  if (n_outer > 0 && (!outer_ids || !inner_mask || !counts))
    return fail(MF_ERR_ARG, "NULL array");
  return cuda_status(
      mf_launch_candidates(*mesh, outer_ids, n_outer, inner_mask, R, reach,
                           counts, nullptr, nullptr, S(stream)),
      "mf_count_candidates");
}

int mf_fill_candidates(const MfMesh *mesh, const int64_t *outer_ids,
                       int64_t n_outer, const uint8_t *inner_mask, int32_t R,
                       double reach, const int64_t *ptr, int64_t *ids,
                       void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (n_outer < 0 || R < 1) return fail(MF_ERR_ARG, "bad n_outer/R");
  if (n_outer == 0) return MF_OK;
  if (!outer_ids || !inner_mask || !ptr) return fail(MF_ERR_ARG, "NULL array");
  if (!ids) {
    // a zero-length ids buffer may be NULL only if there are no pairs;
    // the kernel would not write anything then
    static int64_t dummy;
    ids = &dummy;
  }
  return cuda_status(
      mf_launch_candidates(*mesh, outer_ids, n_outer, inner_mask, R, reach,
                           nullptr, ptr, ids, S(stream)),
      "mf_fill_candidates");
}

size_t mf_scan_workspace_bytes(int64_t n) { return mf_scan_bytes(n); }

int mf_exclusive_scan(const int64_t *counts, int64_t n, int64_t *ptr,
                      void *workspace, size_t ws_bytes, void *stream) {
  if (n < 0 || !ptr || (n > 0 && !counts))
    return fail(MF_ERR_ARG, "bad scan arguments");
  if (n > 0x7fffffffLL) return fail(MF_ERR_UNSUPPORTED, "scan n > 2^31");
  if (n > 0 && ws_bytes < mf_scan_bytes(n))
    return fail(MF_ERR_ARG, "scan workspace too small");
  return cuda_status(mf_scan(counts, n, ptr, workspace, ws_bytes, S(stream)),
                     "mf_exclusive_scan");
}

size_t mf_general_workspace_bytes(const MfMesh *mesh, const MfRules *rules,
                                  int64_t n_inner) {
  (void)mesh;
  int64_t threads = (int64_t)kGenericMaxGrid * kGenericBlock;
  int64_t want = ((n_inner + kGenericBlock - 1) / kGenericBlock) *
                 kGenericBlock;
  if (want < threads) threads = want > 0 ? want : kGenericBlock;
  int nq = rules ? nq_in_max(rules) : 1;
  return (size_t)threads * (size_t)nq * sizeof(double) + 256;
}

int mf_general_core(const MfMesh *mesh, const MfRules *rules,
                    const MfKernel *kern, const MfPattern *pat,
                    const uint8_t *outer_mask, const int32_t *inner_sorted,
                    const int64_t *color_ptr, int32_t ncolors, int32_t R,
                    double scale, double *vals, uint64_t *counters,
                    int32_t flags, void *workspace, size_t ws_bytes,
                    void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (int rc = check_pattern(pat)) return rc;
  if (!rules || !kern) return fail(MF_ERR_ARG, "rules/kernel is NULL");
  if (!color_ptr || ncolors < 1) return fail(MF_ERR_ARG, "bad colours");
  if (!counters || !vals) return fail(MF_ERR_ARG, "vals/counters NULL");
  if (kern->L_min < 1 || kern->L_min > kern->L_max || kern->L_max > 24)
    return fail(MF_ERR_ARG, "need 1 <= L_min <= L_max <= 24");
  if (!(kern->eps >= 0.0 && kern->eps < kern->delta))
    return fail(MF_ERR_ARG, "need 0 <= eps < delta");
  if (R < 1) return fail(MF_ERR_ARG, "R < 1");
  int64_t n_inner = color_ptr[ncolors];
  if (n_inner == 0) return MF_OK;
  if (!outer_mask || !inner_sorted) return fail(MF_ERR_ARG, "NULL masks");
  // vals may be a window pointer shifted before its allocation (multi-GPU
  // row blocks, parallel.py), so only the other arrays are checked
  MF_CHECK_DEV(counters);
  MF_CHECK_DEV(outer_mask);
  MF_CHECK_DEV(inner_sorted);

  AsmParams P = make_params(mesh, rules, kern, pat, outer_mask, R, scale,
                            vals, counters, flags);
  const size_t need = mf_general_workspace_bytes(mesh, rules, n_inner);
  if (!workspace || ws_bytes < need)
    return fail(MF_ERR_ARG, "workspace too small");
  P.overflow = reinterpret_cast<int32_t *>(workspace);
  P.scratch = reinterpret_cast<double *>(static_cast<char *>(workspace) + 256);
  P.scratch_stride = nq_in_max(rules);
  cudaStream_t s = S(stream);

  const bool force_generic = (flags & MF_FLAG_FORCE_GENERIC) != 0;
  const bool tet = (mesh->kinds_present & 8) != 0;
  if (tet && !mf_tet_supported(P))
    // tetrahedra (new element) have one kernel, mf_tet.cu
    return fail(MF_ERR_UNSUPPORTED,
                "tetrahedra need a pure P1 tet mesh, L_max <= 6 and "
                "1/4/11-point tet rules");
  if (mesh->layout != 0 && (mesh->layout != 1 || mesh->row_period < 2))
    return fail(MF_ERR_ARG, "bad mesh layout / row_period");
  // Small structured P1 triangle meshes also take the row-split kernel:
  // their DOFs are lattice ids and an element spans one cell row, so rows
  // two apart share no vertex (row_period 2).  Thread per (element, row)
  // gives 2R+1 times the parallelism of k_2d's thread per element, which
  // leaves the GPU mostly idle below ~10^5 elements (R1: 3,200 elements).
  if (mesh->layout == 0 && mesh->dim == 2 && mesh->kinds_present == 2 &&
      mesh->degree == 1 && mesh->n_elem <= MF_SMALL_TRI_ELEMS &&
      !(flags & MF_FLAG_ELEMENT_THREADS)) {
    AsmParams Q = P;
    Q.mesh.layout = 1;
    Q.mesh.row_period = 2;
    if (!force_generic && mf_tri_u_supported(Q)) P = Q;
  }
  const bool tri_u = !tet && !force_generic && mf_tri_u_supported(P);
  if (tet || tri_u) {
    // row-split kernels (mf_tet.cu planes, mf_2d.cu k_tri_u bin rows):
    // per-row G partials of one colour live in stream-ordered scratch
    // owned by this call (freed on the stream after the last launch)
    int64_t nmax = 0;
    for (int c = 0; c < ncolors; c++)
      nmax = std::max<int64_t>(nmax, color_ptr[c + 1] - color_ptr[c]);
    const size_t nd = tet ? mf_tet_scratch_doubles(P, nmax)
                          : mf_tri_u_scratch_doubles(P, nmax);
    keep_pool();
    double *gscr = nullptr;
    cudaError_t e = cudaMallocAsync(&gscr, sizeof(double) * nd, s);
    if (e != cudaSuccess) return cuda_status(e, "mf_general_core scratch");
    for (int c = 0; c < ncolors && e == cudaSuccess; c++) {
      int64_t n = color_ptr[c + 1] - color_ptr[c];
      if (n <= 0) continue;
      P.inner = inner_sorted + color_ptr[c];
      P.n_inner = n;
      e = tet ? mf_launch_tet(P, gscr, s) : mf_launch_tri_u(P, gscr, s);
    }
    cudaError_t ef = cudaFreeAsync(gscr, s);
    if (e != cudaSuccess) return cuda_status(e, "mf_general_core");
    return cuda_status(ef, "mf_general_core scratch");
  }
  bool use_hex = !force_generic && mf_hex_supported(P);
  bool use_hex2 = use_hex && mf_hex2_supported(P);
  bool use_2d = !force_generic && !use_hex && mf_2d_supported(P);
  for (int c = 0; c < ncolors; c++) {
    int64_t n = color_ptr[c + 1] - color_ptr[c];
    if (n <= 0) continue;
    P.inner = inner_sorted + color_ptr[c];
    P.n_inner = n;
    cudaError_t e;
    if (use_hex2) {
      e = mf_launch_hex2(P, s);
    } else if (use_hex) {
      e = mf_launch_hex(P, s);
    } else if (use_2d) {
      e = mf_launch_2d(P, s);
    } else {
      int64_t want = (n + kGenericBlock - 1) / kGenericBlock;
      int grid = (int)(want < kGenericMaxGrid ? want : kGenericMaxGrid);
      e = mf_launch_generic(P, grid, kGenericBlock, s);
    }
    if (e != cudaSuccess) return cuda_status(e, "mf_general_core");
  }
  return MF_OK;
}

int mf_general_core_lists(const MfMesh *mesh, const MfRules *rules,
                          const MfKernel *kern, const MfPattern *pat,
                          const int64_t *outer_ids, int64_t n_outer,
                          const int64_t *cand_ptr, const int64_t *cand_ids,
                          double scale, double *vals, uint64_t *counters,
                          int32_t flags, void *stream) {
  if (!mesh) return fail(MF_ERR_ARG, "mesh is NULL");
  if (mesh->dim != 2 && mesh->dim != 3) return fail(MF_ERR_ARG, "dim 2/3");
  if (mesh->degree != 1 && mesh->degree != 2)
    return fail(MF_ERR_ARG, "degree must be 1/2");
  if (mesh->n_elem < 0 || mesh->nloc_max < 1)
    return fail(MF_ERR_ARG, "bad mesh sizes");
  if (mesh->n_elem > 0 && (!mesh->elem_kind || !mesh->elem_coords ||
                           !mesh->elem_lo || !mesh->elem_hi ||
                           !mesh->elem_dofs))
    return fail(MF_ERR_ARG, "mesh array is NULL");
  if (int rc = check_pattern(pat)) return rc;
  if (!rules || !kern) return fail(MF_ERR_ARG, "rules/kernel is NULL");
  if (kern->L_min < 1 || kern->L_min > kern->L_max || kern->L_max > 24)
    return fail(MF_ERR_ARG, "need 1 <= L_min <= L_max <= 24");
  if (!(kern->eps >= 0.0 && kern->eps < kern->delta))
    return fail(MF_ERR_ARG, "need 0 <= eps < delta");
  if (n_outer < 0) return fail(MF_ERR_ARG, "n_outer < 0");
  if (!counters || !vals) return fail(MF_ERR_ARG, "vals/counters NULL");
  if (n_outer == 0) return MF_OK;
  if (!outer_ids || !cand_ptr || !cand_ids)
    return fail(MF_ERR_ARG, "NULL list");
  MF_CHECK_DEV(outer_ids);
  MF_CHECK_DEV(cand_ptr);
  MF_CHECK_DEV(cand_ids);
  MF_CHECK_DEV(counters);
  MF_CHECK_DEV(mesh->elem_dofs);
  cudaStream_t s = S(stream);
  // list bounds and outer ids (host checks: the reference has no bounds
  // checks at all, a bad id there is a silent out-of-row write)
  int64_t ends[2];
  cudaError_t e = cudaMemcpyAsync(&ends[0], cand_ptr, 8,
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&ends[1], cand_ptr + n_outer, 8,
                        cudaMemcpyDeviceToHost, s);
  std::vector<int64_t> h_outer(n_outer);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h_outer.data(), outer_ids, 8 * n_outer,
                        cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e, "mf_general_core_lists");
  if (ends[0] != 0 || ends[1] < 0)
    return fail(MF_ERR_ARG, "cand_ptr must start at 0 and be ascending");
  for (int64_t v : h_outer)
    if (v < 0 || v >= mesh->n_elem)
      return fail(MF_ERR_ARG, "outer id out of range");
  const int64_t npairs = ends[1];
  if (npairs == 0) return MF_OK;
  keep_pool();
  MfLists Ls;
  e = mf_lists_build(cand_ptr, cand_ids, outer_ids, n_outer, npairs,
                     mesh->n_elem, mesh->elem_dofs, mesh->nloc_max, s, Ls);
  if (e != cudaSuccess) {
    mf_lists_free(Ls, s);
    if (e == cudaErrorInvalidValue)
      return fail(MF_ERR_ARG, "candidate id out of range");
    return cuda_status(e, "mf_general_core_lists");
  }
  // greedy colouring of the inner elements by shared DOFs (64 colours at
  // most): elements of one colour write disjoint rows, so each colour is
  // one race-free launch (no atomics, deterministic)
  const int64_t n_inner = Ls.n_inner;
  const int nloc = mesh->nloc_max;
  std::vector<uint64_t> used(pat->n, 0);
  std::vector<int> colour(n_inner);
  int ncol = 0;
  for (int64_t t = 0; t < n_inner; t++) {
    uint64_t busy = 0;
    const int64_t *d = Ls.h_dofs.data() + t * nloc;
    for (int j = 0; j < nloc; j++)
      if (d[j] >= 0) {
        if (d[j] >= pat->n) {
          mf_lists_free(Ls, s);
          return fail(MF_ERR_ARG, "element DOF outside the pattern");
        }
        busy |= used[d[j]];
      }
    if (busy == ~0ull) {
      mf_lists_free(Ls, s);
      return fail(MF_ERR_UNSUPPORTED, "more than 64 colours");
    }
    int c = __builtin_ctzll(~busy);
    colour[t] = c;
    ncol = std::max(ncol, c + 1);
    for (int j = 0; j < nloc; j++)
      if (d[j] >= 0) used[d[j]] |= 1ull << c;
  }
  std::vector<int64_t> cptr(ncol + 1, 0), start(n_inner, 0);
  for (int64_t t = 0; t < n_inner; t++) cptr[colour[t] + 1]++;
  for (int c = 0; c < ncol; c++) cptr[c + 1] += cptr[c];
  for (int64_t t = 1; t < n_inner; t++)
    start[t] = start[t - 1] + Ls.h_counts[t - 1];
  std::vector<int32_t> h_inner(n_inner);
  std::vector<int64_t> h_beg(n_inner), h_end(n_inner);
  {
    std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t t = 0; t < n_inner; t++) {
      const int64_t pos = fill[colour[t]]++;
      h_inner[pos] = (int32_t)Ls.h_uniq[t];
      h_beg[pos] = start[t];
      h_end[pos] = start[t] + Ls.h_counts[t];
    }
  }
  int32_t *d_inner = nullptr;
  int64_t *d_be = nullptr;
  double *gscr = nullptr;
  const size_t wsb = mf_general_workspace_bytes(mesh, rules, n_inner);
  e = cudaMallocAsync(&d_inner, 4 * n_inner, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_be, 16 * n_inner, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&gscr, wsb, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(gscr, 0, 256, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_inner, h_inner.data(), 4 * n_inner,
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_be, h_beg.data(), 8 * n_inner,
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_be + n_inner, h_end.data(), 8 * n_inner,
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    AsmParams P = make_params(mesh, rules, kern, pat, nullptr, 1, scale,
                              vals, counters, flags);
    P.overflow = reinterpret_cast<int32_t *>(gscr);
    P.scratch =
        reinterpret_cast<double *>(reinterpret_cast<char *>(gscr) + 256);
    P.scratch_stride = nq_in_max(rules);
    P.list_outer = Ls.list_outer;
    for (int c = 0; c < ncol && e == cudaSuccess; c++) {
      const int64_t n = cptr[c + 1] - cptr[c];
      if (n <= 0) continue;
      P.inner = d_inner + cptr[c];
      P.list_begin = d_be + cptr[c];
      P.list_end = d_be + n_inner + cptr[c];
      P.n_inner = n;
      int64_t want = (n + kGenericBlock - 1) / kGenericBlock;
      int grid = (int)(want < kGenericMaxGrid ? want : kGenericMaxGrid);
      e = mf_launch_generic(P, grid, kGenericBlock, s);
    }
  }
  if (d_inner) cudaFreeAsync(d_inner, s);
  if (d_be) cudaFreeAsync(d_be, s);
  if (gscr) cudaFreeAsync(gscr, s);
  mf_lists_free(Ls, s);
  return cuda_status(e, "mf_general_core_lists");
}

int64_t mf_offset_block_count(int32_t dim, int32_t nproto, int32_t R) {
  const int64_t span = 2 * (int64_t)R + 1;
  return span * span * (dim == 3 ? span : 1) * nproto * nproto;
}

size_t mf_offset_blocks_workspace_bytes(const MfRules *rules, int64_t nblk) {
  const int nq = rules ? nq_in_max(rules) : 1;
  return 256 + (size_t)((nblk + 127) / 128 * 128) * nq * sizeof(double);
}

int mf_offset_blocks(const MfMesh *mesh, const MfRules *rules,
                     const MfKernel *kern, int32_t kind, int32_t nproto,
                     const double *protos, int32_t R, double h, double *B21,
                     double *B22, uint64_t *bev, int32_t flags,
                     void *workspace, size_t ws_bytes, void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (!rules || !kern || !B21 || !B22 || !bev)
    return fail(MF_ERR_ARG, "NULL argument");
  if (kind < 0 || kind > 2 || nproto < 1 || nproto > 2 || R < 1 || !(h > 0))
    return fail(MF_ERR_ARG, "bad block arguments");
  if (kind == 1 && !protos) return fail(MF_ERR_ARG, "protos NULL");
  if (kern->L_min < 1 || kern->L_min > kern->L_max || kern->L_max > 24)
    return fail(MF_ERR_ARG, "need 1 <= L_min <= L_max <= 24");
  const int64_t nblk = mf_offset_block_count(mesh->dim, nproto, R);
  if (!workspace || ws_bytes < mf_offset_blocks_workspace_bytes(rules, nblk))
    return fail(MF_ERR_ARG, "workspace too small");
  AsmParams P = make_params(mesh, rules, kern, nullptr, nullptr, R, 1.0,
                            nullptr, nullptr, flags);
  P.overflow = reinterpret_cast<int32_t *>(workspace);
  P.scratch = reinterpret_cast<double *>(static_cast<char *>(workspace) + 256);
  P.scratch_stride = nq_in_max(rules);
  return cuda_status(
      mf_launch_blocks(P, kind, nproto, R, h, protos, B21, B22,
                       reinterpret_cast<unsigned long long *>(bev), nblk,
                       S(stream)),
      "mf_offset_blocks");
}

int mf_scatter_offset_blocks(const MfMesh *mesh, const MfPattern *pat,
                             int32_t nproto, int32_t R, const int32_t *blk,
                             const int64_t *blk_ptr, const double *B21,
                             const double *B22, const uint64_t *bev,
                             const uint8_t *outer_mask,
                             const int32_t *inner_sorted,
                             const int64_t *color_ptr, int32_t ncolors,
                             double scale, double *vals, uint64_t *counters,
                             void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (int rc = check_pattern(pat)) return rc;
  if (nproto < 1 || nproto > 2 || !blk_ptr || !color_ptr || ncolors < 1)
    return fail(MF_ERR_ARG, "bad scatter arguments");
  if (!vals || !counters || !outer_mask) return fail(MF_ERR_ARG, "NULL");
  const int nloc = mesh->kinds_present == 2
                       ? 3 * mesh->degree
                       : (mesh->dim == 3 ? (mesh->degree + 1) *
                                               (mesh->degree + 1) *
                                               (mesh->degree + 1)
                                         : (mesh->degree + 1) *
                                               (mesh->degree + 1));
  AsmParams P;
  memset(&P, 0, sizeof(P));
  P.mesh = *mesh;
  P.pat = *pat;
  P.outer_mask = outer_mask;
  P.scale = scale;
  P.vals = vals;
  P.counters = reinterpret_cast<unsigned long long *>(counters);
  for (int c = 0; c < ncolors; c++) {
    const int64_t n = color_ptr[c + 1] - color_ptr[c];
    if (n <= 0) continue;
    P.inner = inner_sorted + color_ptr[c];
    P.n_inner = n;
    cudaError_t e = mf_launch_blocked_scatter(
        P, nproto, R, nloc, blk, blk_ptr, B21, B22,
        reinterpret_cast<const unsigned long long *>(bev), S(stream));
    if (e != cudaSuccess) return cuda_status(e, "mf_scatter_offset_blocks");
  }
  return MF_OK;
}

int64_t mf_gather_table_doubles(int32_t dim, int32_t kind, int32_t R);

int mf_offset_block_a22(const MfMesh *mesh, int32_t kind, int32_t nproto,
                        int32_t R, const double *B21, const double *B22,
                        const uint64_t *bev, double *a22, double *table,
                        uint64_t *counters, void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (mesh->degree != 1) return fail(MF_ERR_UNSUPPORTED, "degree 1 only");
  if (kind < 0 || kind > 2 || nproto < 1 || nproto > 2 || R < 1)
    return fail(MF_ERR_ARG, "bad block arguments");
  if (!B21 || !B22 || !bev || !a22 || !table || !counters)
    return fail(MF_ERR_ARG, "NULL");
  MF_CHECK_DEV(a22);
  MF_CHECK_DEV(table);
  AsmParams P;
  memset(&P, 0, sizeof(P));
  P.mesh = *mesh;
  P.counters = reinterpret_cast<unsigned long long *>(counters);
  return cuda_status(
      mf_launch_blocked_a22(
          P, kind, nproto, R, B21, B22,
          reinterpret_cast<const unsigned long long *>(bev), a22, table,
          S(stream)),
      "mf_offset_block_a22");
}

int mf_gather_offset_blocks(const MfMesh *mesh, const MfPattern *pat,
                            int32_t kind, int32_t nproto, int32_t R,
                            const double *table, const double *a22,
                            int64_t row0, int64_t row1, double scale,
                            double *vals, void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (int rc = check_pattern(pat)) return rc;
  if (mesh->degree != 1) return fail(MF_ERR_UNSUPPORTED, "degree 1 only");
  if (row0 < 0 || row1 > pat->n || row0 > row1)
    return fail(MF_ERR_ARG, "bad row range");
  if (!table || !a22 || !vals) return fail(MF_ERR_ARG, "NULL");
  if (pat->K != R + 1) return fail(MF_ERR_ARG, "pattern K != R + 1");
  MF_CHECK_DEV(vals);
  AsmParams P;
  memset(&P, 0, sizeof(P));
  P.mesh = *mesh;
  P.pat = *pat;
  P.scale = scale;
  P.vals = vals;
  keep_pool();
  return cuda_status(mf_launch_blocked_gather(P, kind, nproto, R, table,
                                              a22, row0, row1, S(stream)),
                     "mf_gather_offset_blocks");
}

int mf_scale(double *vals, int64_t nnz, double sc, void *stream) {
  if (nnz < 0 || (nnz > 0 && !vals)) return fail(MF_ERR_ARG, "bad scale");
  return cuda_status(mf_launch_scale(vals, nnz, sc, S(stream)), "mf_scale");
}

int mf_asymmetry_inf(const MfPattern *pat, const double *vals, double *out,
                     void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !out) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(out);
  return cuda_status(mf_launch_asym(*pat, vals, out, S(stream)),
                     "mf_asymmetry_inf");
}

int mf_asymmetry_inf_rows(const MfPattern *pat, const double *vals,
                          int64_t row0, int64_t row1, double *out,
                          void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !out) return fail(MF_ERR_ARG, "NULL array");
  if (row0 < 0 || row1 > pat->n || row0 > row1)
    return fail(MF_ERR_ARG, "bad row range");
  MF_CHECK_DEV(out);
  return cuda_status(mf_launch_asym_rows(*pat, vals, row0, row1, out,
                                         S(stream)),
                     "mf_asymmetry_inf_rows");
}

int mf_norm_inf(const MfPattern *pat, const double *vals, double *out,
                void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !out) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(out);
  return cuda_status(mf_launch_norm(*pat, vals, out, S(stream)),
                     "mf_norm_inf");
}

int mf_matvec(const MfPattern *pat, const double *vals, const double *x,
              double *y, void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !x || !y) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(x);
  MF_CHECK_DEV(y);
  return cuda_status(mf_launch_matvec(*pat, vals, x, y, S(stream)),
                     "mf_matvec");
}

int mf_diag(const MfPattern *pat, const double *vals, double *out,
            void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !out) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(out);
  return cuda_status(mf_launch_diag(*pat, vals, out, S(stream)), "mf_diag");
}

int mf_symmetrize(const MfPattern *pat, double *vals, void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  return cuda_status(mf_launch_symmetrize(*pat, vals, S(stream)),
                     "mf_symmetrize");
}

int mf_fill_cols(const MfPattern *pat, int64_t *cols, void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!cols) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(cols);
  return cuda_status(mf_launch_fill_cols(*pat, cols, S(stream)),
                     "mf_fill_cols");
}

int mf_load_scatter(const MfMesh *mesh, const int32_t *elems,
                    const int64_t *color_ptr, int32_t ncolors,
                    const double *fval, const double *w, const double *phi,
                    int32_t nq, int32_t nloc, double *load, void *stream) {
  if (int rc = check_mesh(mesh)) return rc;
  if (!color_ptr || ncolors < 1 || nq < 1 || nloc < 1 ||
      nloc > mesh->nloc_max)
    return fail(MF_ERR_ARG, "bad load arguments");
  if (color_ptr[ncolors] > 0 && (!elems || !fval || !w || !phi || !load))
    return fail(MF_ERR_ARG, "NULL array");
  for (int c = 0; c < ncolors; c++) {
    const int64_t a = color_ptr[c], n = color_ptr[c + 1] - a;
    if (n <= 0) continue;
    cudaError_t e = mf_launch_load(*mesh, elems + a, n, fval + a * nq, w, phi,
                                   nq, nloc, load, S(stream));
    if (e != cudaSuccess) return cuda_status(e, "mf_load_scatter");
  }
  return MF_OK;
}

size_t mf_vec_workspace_bytes(void) { return mf_vec_ws_bytes(); }

int mf_cg_matvec_dot(const MfPattern *pat, const double *vals,
                     const double *p, const uint8_t *cmask, double *Ap,
                     double *out, void *ws, void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !p || !cmask || !Ap || !out || !ws)
    return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(Ap);
  return cuda_status(
      mf_launch_cg_matvec_dot(*pat, vals, p, cmask, Ap, out,
                              static_cast<double *>(ws), S(stream)),
      "mf_cg_matvec_dot");
}

int mf_cg_update(int64_t n, double alpha, const double *p, const double *Ap,
                 const double *dinv, double *x, double *r, double *z,
                 double *out, void *ws, void *stream) {
  if (n < 0 || (n > 0 && (!p || !Ap || !dinv || !x || !r || !z)) || !out ||
      !ws)
    return fail(MF_ERR_ARG, "bad cg update arguments");
  return cuda_status(mf_launch_cg_update(n, alpha, p, Ap, dinv, x, r, z, out,
                                         static_cast<double *>(ws),
                                         S(stream)),
                     "mf_cg_update");
}

int mf_cg_direction(int64_t n, double beta, const double *z, double *p,
                    void *stream) {
  if (n < 0 || (n > 0 && (!z || !p)))
    return fail(MF_ERR_ARG, "bad cg direction arguments");
  return cuda_status(mf_launch_cg_direction(n, beta, z, p, S(stream)),
                     "mf_cg_direction");
}

int mf_jacobi_inverse(int64_t n, const double *diag, const uint8_t *cmask,
                      double *dinv, double *out_min_free, void *ws,
                      void *stream) {
  if (n < 0 || (n > 0 && (!diag || !cmask || !dinv)) || !out_min_free || !ws)
    return fail(MF_ERR_ARG, "bad jacobi arguments");
  return cuda_status(mf_launch_jacobi(n, diag, cmask, dinv, out_min_free,
                                      static_cast<double *>(ws), S(stream)),
                     "mf_jacobi_inverse");
}

int mf_gather_diff(int64_t n_sel, const int64_t *idx, const double *a,
                   const double *b, double *out, void *stream) {
  if (n_sel < 0 || (n_sel > 0 && (!idx || !a || !out)))
    return fail(MF_ERR_ARG, "bad gather arguments");
  return cuda_status(mf_launch_gather_diff(n_sel, idx, a, b, out, S(stream)),
                     "mf_gather_diff");
}

int mf_scatter_values(int64_t n_sel, const int64_t *idx, const double *v,
                      double *out, void *stream) {
  if (n_sel < 0 || (n_sel > 0 && (!idx || !v || !out)))
    return fail(MF_ERR_ARG, "bad scatter arguments");
  return cuda_status(mf_launch_scatter(n_sel, idx, v, out, S(stream)),
                     "mf_scatter_values");
}

int mf_sum_ordered(int32_t nbuf, const double *const *bufs, int64_t n,
                   double scale, double *out, void *stream) {
  if (nbuf < 1 || nbuf > 64 || !bufs || n < 0 || (n > 0 && !out))
    return fail(MF_ERR_ARG, "bad buffer-sum arguments");
  for (int k = 0; k < nbuf; k++)
    if (n > 0 && !bufs[k]) return fail(MF_ERR_ARG, "NULL buffer");
  return cuda_status(mf_launch_sum_ordered(nbuf, bufs, n, scale, out,
                                           S(stream)),
                     "mf_sum_ordered");
}

int mf_row_touched(const MfPattern *pat, const double *vals, uint8_t *flags,
                   void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !flags) return fail(MF_ERR_ARG, "NULL array");
  MF_CHECK_DEV(vals);
  MF_CHECK_DEV(flags);
  return cuda_status(mf_launch_row_touched(*pat, vals, flags, S(stream)),
                     "mf_row_touched");
}

int mf_axpby(int64_t n, double a, const double *x, double b,
             const double *y, double *out, void *stream) {
  if (n < 0 || (n > 0 && (!x || !y || !out)))
    return fail(MF_ERR_ARG, "bad axpby arguments");
  return cuda_status(mf_launch_axpby(n, a, x, b, y, out, S(stream)),
                     "mf_axpby");
}

int mf_matvec_rows(const MfPattern *pat, const double *vals, const double *x,
                   int64_t row0, int64_t row1, double *y, void *stream) {
  if (int rc = check_pattern(pat)) return rc;
  if (!vals || !x || !y) return fail(MF_ERR_ARG, "NULL array");
  if (row0 < 0 || row1 > pat->n || row0 > row1)
    return fail(MF_ERR_ARG, "bad row range");
  MF_CHECK_DEV(x);
  MF_CHECK_DEV(y);
  return cuda_status(mf_launch_matvec_rows(*pat, vals, x, row0, row1, y,
                                           S(stream)),
                     "mf_matvec_rows");
}

int mf_fp64_probe(double *out, int64_t iters, int32_t blocks,
                  int32_t threads, void *stream) {
  if (!out || iters < 1 || blocks < 1 || threads < 32 || threads > 1024)
    return fail(MF_ERR_ARG, "bad probe arguments");
  return cuda_status(mf_launch_probe(out, iters, blocks, threads, S(stream)),
                     "mf_fp64_probe");
}

double mf_fp64_probe_flops(int64_t iters, int32_t blocks, int32_t threads) {
  return 2.0 * 8.0 * (double)iters * (double)blocks * (double)threads;
}

}  // extern "C"
