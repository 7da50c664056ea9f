/*
 * mollifem_b200.h -- C-ABI of the B200 nonlocal stiffness assembly.
 *
 * Drop-in replacement for the numba cores the reference package binds on
 * its hot path (/root/reference/pkg/src/mollifem/_kernels.py).  Plain C:
 * pointers, sizes and an opaque stream handle; no torch or CUDA types.
 *
 * Conventions:
 *   - every array argument is caller-owned DEVICE memory unless the
 *     parameter comment says "host";
 *   - kernels accumulate in place into `vals` like the reference cores;
 *   - return 0 on success, MF_ERR_* otherwise; mf_last_error() gives a
 *     thread-local message;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - no global mutable state: calls on distinct streams/devices with
 *     disjoint output buffers may run concurrently.
 */
#ifndef MOLLIFEM_B200_H
#define MOLLIFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_OK 0
#define MF_ERR_ARG 1
#define MF_ERR_CUDA 2
#define MF_ERR_UNSUPPORTED 3

#define MF_ABI_VERSION 3

/* Mesh SoA + DOF map (mesh.py:78-88 flat arrays; fe_space.py:131-157). */
typedef struct MfMesh {
  int32_t dim;              /* 2 or 3 */
  int32_t degree;           /* FE degree 1 or 2 */
  int64_t n_elem;
  int32_t nv_max;           /* geometry rows per element in elem_coords */
  int32_t nloc_max;         /* columns of elem_dofs */
  const int8_t *elem_kind;  /* (n) 0 quad, 1 tri, 2 hex */
  const double *elem_coords;/* (n, nv_max, dim) */
  const double *elem_lo;    /* (n, dim) bounding boxes */
  const double *elem_hi;    /* (n, dim) */
  const int64_t *elem_dofs; /* (n, nloc_max), -1 padded */
  const int32_t *elem_cell; /* (n) flat cell id, x fastest (assembly.py:135) */
  const int64_t *cell_ptr;  /* (ncells+1) elements per cell, cell-lex order */
  int32_t ncx, ncy, ncz;    /* cell grid (ncz = 1 in 2D) */
  int32_t kinds_present;    /* bit k set if some element has kind k */
  /* 0: the reference's structured layout (elements in cell-lex order,
   *    DOFs from cell + proto offsets).
   * 1: unstructured P1 triangles (new, BASELINE config #2): elements in
   *    the bin of their box lower corner, any shape; elem_dofs are lattice
   *    ids on the pattern grid.  Outer elements binned row_period rows
   *    apart share no vertex (the kernel splits the stencil rows into
   *    row_period race-free classes). */
  int32_t layout;
  int32_t row_period;
} MfMesh;

/* Reference-element rules and inner shape tables (assembly.py:333-356).
 * Tensor box rules also pass their 1D factor (n1d points/weights) so the
 * specialised kernels can sum-factorise; n1d = 0 disables that path. */
typedef struct MfRules {
  int32_t nq_box_out, nq_box_in, nq_tri_out, nq_tri_in;
  const double *box_out_pts, *box_out_w;  /* (nq, dim), (nq) */
  const double *box_in_pts, *box_in_w;
  /* simplex slots: triangles (nq, 2) in 2D; in 3D the tetrahedron rule
   * (nq, 3) of the P1 tet element (new; mesh kind 3, kinds_present bit 8) */
  const double *tri_out_pts, *tri_out_w;  /* (nq, dim), (nq) */
  const double *tri_in_pts, *tri_in_w;
  const double *phi_box_in;               /* (nq_box_in, nl_box) */
  const double *phi_tri_in;               /* (nq_tri_in, nl_tri); nl = 4 for tets */
  int32_t n1d_box_out, n1d_box_in;
  const double *box_out_x1d, *box_out_w1d;/* (n1d) */
  const double *box_in_x1d, *box_in_w1d;
} MfRules;

/* Kernel + Algorithm-1 parameters (kernel.py:114-152, assembly.py:51-83). */
typedef struct MfKernel {
  double delta, eps, cde;   /* cde = C_{delta,eps} */
  int32_t L_min, L_max;
} MfKernel;

/* Implicit structured pattern (assembly.py:189-223, 313-327): row r holds
 * the clipped grid box of half-width K around r, x fastest. */
typedef struct MfPattern {
  int32_t NX, NY, NZ, K;
  int64_t n;                /* rows = n_dofs */
  const int64_t *rowptr;    /* (n+1) */
} MfPattern;

/* Counter slots written by mf_general_core (device uint64[MF_NCOUNTERS]). */
#define MF_CNT_EVENTS 0        /* integration events (== reference events) */
#define MF_CNT_PAIRS 1         /* (outer, inner) pairs visited */
#define MF_CNT_EV_UPPER 2      /* events at level < L_max (mu == 1 plateau) */
#define MF_CNT_EV_PLATEAU 3    /* L_max events proven inside delta-eps */
#define MF_CNT_EV_DEAD 4       /* L_max events proven beyond delta+eps */
#define MF_CNT_EV_FULL 5       /* L_max events integrated point by point */
#define MF_CNT_OVERFLOW 6      /* nonzero: a specialised kernel dropped
                                  work it could not hold (more split nodes
                                  per level than it buffers); the values
                                  are incomplete and the caller must treat
                                  the call as failed (MF_ERR_UNSUPPORTED) */
#define MF_NCOUNTERS 10        /* slots 7-9: debug statistics builds */

/* Neighbour search.  Replaces _count_candidates/_fill_candidates
 * (_kernels.py:1205-1268) as driven by _candidates (assembly.py:157-175):
 * for outer element outer_ids[i], the inner elements e with inner_mask[e]
 * in the (2R+1)^dim cell stencil whose max-axis box gap is < reach, in
 * ascending id order.  Bit-exact with the reference. */
int mf_count_candidates(const MfMesh *mesh, const int64_t *outer_ids,
                        int64_t n_outer, const uint8_t *inner_mask,
                        int32_t R, double reach, int64_t *counts,
                        void *stream);
int mf_fill_candidates(const MfMesh *mesh, const int64_t *outer_ids,
                       int64_t n_outer, const uint8_t *inner_mask,
                       int32_t R, double reach, const int64_t *ptr,
                       int64_t *ids, void *stream);

/* ptr[0] = 0, ptr[i+1] = sum(counts[0..i]) (np.cumsum, assembly.py:169). */
size_t mf_scan_workspace_bytes(int64_t n);
int mf_exclusive_scan(const int64_t *counts, int64_t n, int64_t *ptr,
                      void *workspace, size_t ws_bytes, void *stream);

/* Adaptive pair assembly.  Replaces _general_core (_kernels.py:391-487)
 * together with the candidate lists it consumes: every pair (l, m) with
 * outer_mask[l], m in inner_sorted and max-axis box gap < delta+eps runs
 * Algorithm 1 (_pair_blocks, _kernels.py:184-313) with bit-exact
 * classification; scale*(A21 + A22) blocks are added into vals (scale = 2
 * folds _finish's doubling, assembly.py:441).
 *
 * inner_sorted (device int32) lists the inner elements grouped by colour;
 * color_ptr (HOST int64[ncolors+1]) delimits the groups.  Elements of one
 * colour share no DOF, so each colour is one race-free, atomic-free launch
 * and the result is deterministic.  counters: device uint64[MF_NCOUNTERS]
 * (accumulated).  flags: MF_FLAG_* below.  workspace: device scratch of at
 * least mf_general_workspace_bytes() bytes. */
#define MF_FLAG_FORCE_GENERIC 1   /* bypass the specialised kernels */
#define MF_FLAG_NO_SHORTCUTS 2    /* integrate proven-plateau/dead events
                                     point by point too */
#define MF_FLAG_ELEMENT_THREADS 4 /* small structured P1 triangle meshes:
                                     keep the thread-per-element kernel
                                     instead of the row-split one */
#define MF_FLAG_HEX_LEVELS 8      /* hex Q1 meshes with L_max == 2: keep the
                                     level-synchronous kernel (k_hex) instead
                                     of the separable one (k_hex2) */
size_t mf_general_workspace_bytes(const MfMesh *mesh, const MfRules *rules,
                                  int64_t n_inner);
int mf_general_core(const MfMesh *mesh, const MfRules *rules,
                    const MfKernel *kern, const MfPattern *pat,
                    const uint8_t *outer_mask, const int32_t *inner_sorted,
                    const int64_t *color_ptr, int32_t ncolors, int32_t R,
                    double scale, double *vals, uint64_t *counters,
                    int32_t flags, void *workspace, size_t ws_bytes,
                    void *stream);

/* Explicit candidate lists: the exact argument form of _general_core
 * (_kernels.py:391-400).  For i < n_outer and k in [cand_ptr[i],
 * cand_ptr[i+1]) the pair (outer_ids[i], cand_ids[k]) runs Algorithm 1 --
 * every listed pair, with no gap test, duplicates counted twice, as the
 * reference does -- and scale*(A21 + A22) is added into vals.  All four
 * list arrays are device memory (int64); cand_ptr[0] must be 0.  The lists
 * are transposed on the device to per-inner-element ranges (stable radix
 * sort: each inner element keeps the caller's pair order), the inner
 * elements are coloured greedily by shared DOFs on the host (at most 64
 * colours) and each colour runs as one race-free launch of the generic
 * kernel.  Only elem_kind/coords/lo/hi/dofs of the mesh are read (the cell
 * grid may be NULL).  Synchronises `stream` (the list sizes are read back);
 * scratch is stream-ordered (cudaMallocAsync).  The product-form pair sets
 * that _run_general builds (outer ids x inner mask, gap < delta+eps) are
 * faster through mf_general_core, which runs the specialised kernels. */
int mf_general_core_lists(const MfMesh *mesh, const MfRules *rules,
                          const MfKernel *kern, const MfPattern *pat,
                          const int64_t *outer_ids, int64_t n_outer,
                          const int64_t *cand_ptr, const int64_t *cand_ids,
                          double scale, double *vals, uint64_t *counters,
                          int32_t flags, void *stream);

/* Offset-blocked strategy, the reference default on pure meshes
 * (strategy "auto"/"blocked", assembly.py:391-437).  mf_offset_blocks runs
 * Algorithm 1 once per (cell offset d in [-R,R]^dim, outer proto t2, inner
 * proto t1) on the reference's synthetic geometry (_build_offset_blocks,
 * _kernels.py:490-594); block bi = (((dz*S + dy)*S + dx)*np + t2)*np + t1
 * with S = 2R+1 (offsets shifted by R), B21/B22 are (nblk, nloc, nloc),
 * bev the per-block event count (0 = absent block).  protos: device
 * (nproto, 3, 2) triangle protos in cell units (NULL for boxes).
 * mf_scatter_offset_blocks adds every realised (inner element, block)
 * (_scatter_offset_blocks, _kernels.py:597-647): blk lists the present
 * blocks grouped by inner proto, blk_ptr (HOST int64[nproto+1]) delimits
 * the groups; A22 blocks are summed per inner element; counters get the
 * realised events and pairs. */
int64_t mf_offset_block_count(int32_t dim, int32_t nproto, int32_t R);
size_t mf_offset_blocks_workspace_bytes(const MfRules *rules, int64_t nblk);
int mf_offset_blocks(const MfMesh *mesh, const MfRules *rules,
                     const MfKernel *kern, int32_t kind, int32_t nproto,
                     const double *protos, int32_t R, double h, double *B21,
                     double *B22, uint64_t *bev, int32_t flags,
                     void *workspace, size_t ws_bytes, void *stream);
int mf_scatter_offset_blocks(const MfMesh *mesh, const MfPattern *pat,
                             int32_t nproto, int32_t R, const int32_t *blk,
                             const int64_t *blk_ptr, const double *B21,
                             const double *B22, const uint64_t *bev,
                             const uint8_t *outer_mask,
                             const int32_t *inner_sorted,
                             const int64_t *color_ptr, int32_t ncolors,
                             double scale, double *vals, uint64_t *counters,
                             void *stream);

/* Gather form of the blocked scatter (degree 1 only).
 * mf_offset_block_a22 re-lays the present B21 blocks into the gather
 * table (device scratch of mf_gather_table_doubles() doubles: the block
 * entries with the cell offset innermost, zero-padded), sums every
 * element's realised B22 blocks into a22 (n_elem, nloc, nloc) and adds the
 * realised events/pairs to counters.  mf_gather_offset_blocks then WRITES
 * (not adds) vals for rows [row0, row1): entry (r, c) is the sum over
 * inner m containing r and outer l containing c of the present block of
 * offset cell(m) - cell(l), plus a22 of m when c is a DOF of m -- the sum
 * _scatter_offset_blocks accumulates, computed entry by entry (coalesced,
 * deterministic, no read-modify-write). */
int64_t mf_gather_table_doubles(int32_t dim, int32_t kind, int32_t R);
int mf_offset_block_a22(const MfMesh *mesh, int32_t kind, int32_t nproto,
                        int32_t R, const double *B21, const double *B22,
                        const uint64_t *bev, double *a22, double *table,
                        uint64_t *counters, void *stream);
int mf_gather_offset_blocks(const MfMesh *mesh, const MfPattern *pat,
                            int32_t kind, int32_t nproto, int32_t R,
                            const double *table, const double *a22,
                            int64_t row0, int64_t row1, double scale,
                            double *vals, void *stream);

/* Matrix utilities on the implicit pattern (_kernels.py:846-1202). */
int mf_scale(double *vals, int64_t nnz, double s, void *stream);
/* out: device double[1]; max over rows of sum_c |A_rc - A_cr| */
int mf_asymmetry_inf(const MfPattern *pat, const double *vals, double *out,
                     void *stream);
/* the same over rows [row0, row1) only: vals may be a window pointer
 * (shifted by its base) holding every row within K grid planes of the
 * range (distributed row blocks, parallel.py) */
int mf_asymmetry_inf_rows(const MfPattern *pat, const double *vals,
                          int64_t row0, int64_t row1, double *out,
                          void *stream);
int mf_norm_inf(const MfPattern *pat, const double *vals, double *out,
                void *stream);
int mf_matvec(const MfPattern *pat, const double *vals, const double *x,
              double *y, void *stream);
int mf_diag(const MfPattern *pat, const double *vals, double *out,
            void *stream);
int mf_symmetrize(const MfPattern *pat, double *vals, void *stream);
int mf_fill_cols(const MfPattern *pat, int64_t *cols, void *stream);

/* Load vector (assemble_rhs's _group_load, assembly.py:641-676): for each
 * element e = elems[k] (colour-grouped like mf_general_core; color_ptr is
 * HOST memory), load[dofs[e,i]] += |J_e| sum_q fval[k*nq + q] w[q] phi[q,i]
 * with |J| = det (triangles) or prod 0.5*(hi-lo) (boxes).  fval holds the
 * caller's f at the physical rule points of elements[k] (host callables
 * are evaluated by the caller).  All elements must share one kind. */
int mf_load_scatter(const MfMesh *mesh, const int32_t *elems,
                    const int64_t *color_ptr, int32_t ncolors,
                    const double *fval, const double *w, const double *phi,
                    int32_t nq, int32_t nloc, double *load, void *stream);

/* Device solver and glue (solver.py:26-90, assembly.py:679-691,
 * parallel.py:180-200).  Reductions are deterministic (fixed grid, block
 * partials summed in block order); ws: device scratch of at least
 * mf_vec_workspace_bytes() bytes; every out is a device double array.
 *   mf_cg_matvec_dot  Ap = A p with rows where cmask != 0 zeroed;
 *                     out[0] = p.Ap
 *   mf_cg_update      x += alpha p; r -= alpha Ap; z = dinv r;
 *                     out[0] = r.r, out[1] = r.z
 *   mf_cg_direction   p = z + beta p
 *   mf_jacobi_inverse dinv = cmask ? 0 : 1/diag; out[0] = min free diag
 *   mf_gather_diff    out[k] = a[idx[k]] - b[idx[k]] (b may be NULL)
 *   mf_scatter_values out[idx[k]] = v[k]
 *   mf_sum_ordered    out = scale * (bufs[0] + bufs[1] + ...) summed in
 *                     buffer order (bufs: HOST array of <= 64 device
 *                     pointers)
 *   mf_row_touched    flags[r] = row r holds a nonzero value */
size_t mf_vec_workspace_bytes(void);
int mf_cg_matvec_dot(const MfPattern *pat, const double *vals,
                     const double *p, const uint8_t *cmask, double *Ap,
                     double *out, void *ws, void *stream);
int mf_cg_update(int64_t n, double alpha, const double *p, const double *Ap,
                 const double *dinv, double *x, double *r, double *z,
                 double *out, void *ws, void *stream);
int mf_cg_direction(int64_t n, double beta, const double *z, double *p,
                    void *stream);
int mf_jacobi_inverse(int64_t n, const double *diag, const uint8_t *cmask,
                      double *dinv, double *out_min_free, void *ws,
                      void *stream);
int mf_gather_diff(int64_t n_sel, const int64_t *idx, const double *a,
                   const double *b, double *out, void *stream);
int mf_scatter_values(int64_t n_sel, const int64_t *idx, const double *v,
                      double *out, void *stream);
int mf_sum_ordered(int32_t nbuf, const double *const *bufs, int64_t n,
                   double scale, double *out, void *stream);
int mf_row_touched(const MfPattern *pat, const double *vals, uint8_t *flags,
                   void *stream);
/* out = a x + b y (out may alias x or y) */
int mf_axpby(int64_t n, double a, const double *x, double b,
             const double *y, double *out, void *stream);
/* y[r] = (A x)[r] for rows [row0, row1) only; vals may be a window
 * pointer holding those rows (distributed row blocks) */
int mf_matvec_rows(const MfPattern *pat, const double *vals, const double *x,
                   int64_t row0, int64_t row1, double *y, void *stream);

/* FP64 roofline probe: independent DFMA chains; out = device double[1]
 * (sink).  Time it with events to get the sustained DFMA rate. */
int mf_fp64_probe(double *out, int64_t iters, int32_t blocks,
                  int32_t threads, void *stream);
/* flops executed by one mf_fp64_probe launch with these arguments */
double mf_fp64_probe_flops(int64_t iters, int32_t blocks, int32_t threads);

const char *mf_last_error(void);
int mf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif
