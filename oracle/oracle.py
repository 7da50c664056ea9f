"""ctypes front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  It wraps
``oracle/build/libmf_oracle.so`` (built from ``mf_oracle.c`` by
``oracle/Makefile``), the C restatement of the reference numba cores
(/root/reference/pkg/src/mollifem/_kernels.py), and mirrors the reference
entry points that drive them:

  candidates()        assembly.py:157-175   (_candidates)
  run_general()       assembly.py:369-388   (_run_general -> _general_core)
  assemble_general()  assembly.py:456-473   (assemble, strategy="general")
  asymmetry_inf(), matvec(), diag(), symmetrize()  _kernels.py:871-1202

Inputs (mesh arrays, rules, shape tables) come from the product package's
host layer, which tests/test_host_layer.py pins bit-identical to the
reference's.  The oracle itself is pinned against the live reference by the
golden fixtures in tests/golden (tests/test_oracle_golden.py).
"""

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libmf_oracle.so")
_lib = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_GENERAL = ([C.c_int, C.c_int, _i8p, _f64p, C.c_int, _f64p, _f64p, _i64p,
             C.c_int, _i64p, C.c_int64, _i64p, _i64p]
            + [_f64p, _f64p, C.c_int] * 4
            + [_f64p, _f64p, C.c_double, C.c_double, C.c_double, C.c_int,
               C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i64p])


def build():
    """Compile the oracle library (gcc, no FMA contraction)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        build()
    L = C.CDLL(_LIB_PATH)
    L.orc_general_core.restype = C.c_int64
    L.orc_general_core.argtypes = _GENERAL + [C.c_void_p, C.c_void_p]
    L.orc_general_core_mt.restype = C.c_int64
    L.orc_general_core_mt.argtypes = _GENERAL + [C.POINTER(C.c_void_p),
                                                 C.c_int, C.c_int64]
    cand = [_i64p, C.c_int64, _i32p, _f64p, _f64p, _u8p, _i64p, C.c_int,
            C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
    L.orc_count_candidates.restype = None
    L.orc_count_candidates.argtypes = cand + [_i64p]
    L.orc_fill_candidates.restype = None
    L.orc_fill_candidates.argtypes = cand + [_i64p, _i64p]
    pat = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64]
    L.orc_asymmetry_inf.restype = C.c_double
    L.orc_asymmetry_inf.argtypes = [_i64p, _f64p] + pat
    L.orc_matvec.restype = None
    L.orc_matvec.argtypes = [_i64p, _f64p, _f64p, _f64p] + pat
    L.orc_symmetrize.restype = None
    L.orc_symmetrize.argtypes = [_i64p, _f64p] + pat
    L.orc_diag.restype = None
    L.orc_diag.argtypes = [_i64p, _f64p, C.c_int, C.c_int, C.c_int,
                           C.c_int64, _f64p]
    _lib = L
    return L


def _grid(mesh):
    nc = mesh.grid_ncells
    return int(nc[0]), int(nc[1]), int(nc[2]) if mesh.dim == 3 else 1


def candidates(mesh, reach, outer_ids, inner_mask):
    """(ptr, ids) exactly as the reference `_candidates`."""
    from paper_2101_08825_b200.assembly import stencil_pad, stencil_radius
    L = lib()
    flat, cptr = mesh.cell_ptr()
    ncx, ncy, ncz = _grid(mesh)
    R = stencil_radius(reach + stencil_pad(mesh), mesh.h)
    outer = np.ascontiguousarray(outer_ids, dtype=np.int64)
    mask = np.ascontiguousarray(inner_mask, dtype=np.uint8)
    counts = np.empty(len(outer), dtype=np.int64)
    args = (outer, len(outer), flat, mesh.elem_lo, mesh.elem_hi, mask, cptr,
            ncx, ncy, ncz, R, mesh.dim, float(reach))
    L.orc_count_candidates(*args, counts)
    ptr = np.zeros(len(outer) + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    ids = np.empty(int(ptr[-1]), dtype=np.int64)
    L.orc_fill_candidates(*args, ptr, ids)
    return ptr, ids


def _general_args(mesh, space, params, config, outer, ptr, ids, A, P=None):
    from paper_2101_08825_b200.assembly import prep_tables
    if P is None:
        P = prep_tables(mesh, space, config)
    return (mesh.dim, space.degree, mesh.elem_kind, mesh.elem_coords,
            mesh.elem_coords.shape[1], mesh.elem_lo, mesh.elem_hi,
            space.element_dofs, space.element_dofs.shape[1], outer,
            len(outer), ptr, ids,
            P.box_out_pts, P.box_out_w, len(P.box_out_w),
            P.box_in_pts, P.box_in_w, len(P.box_in_w),
            P.tri_out_pts, P.tri_out_w, len(P.tri_out_w),
            P.tri_in_pts, P.tri_in_w, len(P.tri_in_w),
            P.PHI_box_in, P.PHI_tri_in,
            params.delta, params.eps, params.c_delta_eps,
            config.L_min, config.L_max, A.NX, A.NY, A.NZ, A.K, A.rowptr)


def run_general(mesh, space, params, config, A, outer_ids=None,
                inner_mask=None, census=None):
    """`_run_general` (assembly.py:369-388): accumulate into A.vals (host).

    census: optional int64[7] (see mf_oracle.c orc_general_core)."""
    n = mesh.n_elements
    outer = (np.arange(n, dtype=np.int64) if outer_ids is None
             else np.ascontiguousarray(outer_ids, dtype=np.int64))
    mask = (np.ones(n, dtype=np.uint8) if inner_mask is None
            else np.ascontiguousarray(inner_mask, dtype=np.uint8))
    ptr, ids = candidates(mesh, params.delta + params.eps, outer, mask)
    args = _general_args(mesh, space, params, config, outer, ptr, ids, A)
    cen = None if census is None else census.ctypes.data_as(C.c_void_p)
    return int(lib().orc_general_core(
        *args, np.ascontiguousarray(A.vals).ctypes.data_as(C.c_void_p), cen))


def run_general_threads(mesh, space, params, config, A, outer_ids,
                        nthreads, private=True, blk=4):
    """Threaded timing driver over disjoint outer subsets.

    private=True gives every thread its own zeroed copy of A.vals and sums
    them into A.vals afterwards (the reference's parallel_assemble buffers,
    parallel.py:157-200); private=False shares A.vals (timing only: the
    unsynchronised adds may lose updates, values are not used).
    Returns (events, seconds_compute)."""
    import time
    outer = np.ascontiguousarray(outer_ids, dtype=np.int64)
    mask = np.ones(mesh.n_elements, dtype=np.uint8)
    ptr, ids = candidates(mesh, params.delta + params.eps, outer, mask)
    args = _general_args(mesh, space, params, config, outer, ptr, ids, A)
    bufs = ([np.zeros_like(A.vals) for _ in range(nthreads)] if private
            else [A.vals] * nthreads)
    arr = (C.c_void_p * nthreads)(*[b.ctypes.data for b in bufs])
    t0 = time.perf_counter()
    ev = int(lib().orc_general_core_mt(*args, arr, nthreads, blk))
    dt = time.perf_counter() - t0
    if private:
        for b in bufs:
            A.vals += b
    return ev, dt


def run_general_tiled(mesh, space, params, config, pat, inner_ids, vals,
                      base=0, nthreads=None, tile=None):
    """`_run_general(outer_ids=all, inner_mask=inner_ids)` on host threads.

    The inner elements are cut into tiles of `tile`^dim cells; tiles whose
    tile coordinates have the same parity bits share no DOF (an element of
    cell c only touches DOF planes [d*c, d*(c+1)] per axis), so each parity
    class runs its tiles concurrently (ctypes releases the GIL) into ONE
    value array without races, and the classes run one after another.
    Every pair is evaluated by orc_general_core exactly as the serial call
    would and each value entry receives its pair blocks in a fixed order
    (parity class, then tile, then the serial order), so the result does
    not depend on the thread count; it equals the serial run up to the
    summation order of entries shared by tiles (rounding level).

    pat: a HostPattern (rowptr, grid); vals: float64 array holding the
    pattern's entries [base, base + len(vals)) -- a window is enough when
    the inner elements' rows lie inside it.  Returns the event count."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2101_08825_b200.assembly import stencil_pad, stencil_radius
    L = lib()
    n = mesh.n_elements
    dim = mesh.dim
    inner = np.ascontiguousarray(inner_ids, dtype=np.int64)
    reach = params.delta + params.eps
    R = stencil_radius(reach + stencil_pad(mesh), mesh.h)
    cell = np.asarray(mesh.elem_cell, dtype=np.int64)[:, :dim]
    if tile is None:
        # Delaunay vertices may sit dof_spill planes above their bin
        tile = max(2, int(getattr(mesh, "dof_spill", 1)) + 1)
    tc = cell[inner] // tile
    colour = np.zeros(len(inner), dtype=np.int64)
    for k in range(dim):
        colour |= (tc[:, k] & 1) << k
    key = np.zeros(len(inner), dtype=np.int64)
    for k in range(dim):
        key = key * (int(tc[:, k].max()) + 1 if len(inner) else 1) + tc[:, k]
    assert vals.dtype == np.float64 and vals.flags.c_contiguous
    vptr = vals.ctypes.data - 8 * int(base)
    PT = prep_tables_cached(mesh, space, config)

    def run_tile(elems):
        lo = cell[elems].min(axis=0) - R
        hi = cell[elems].max(axis=0) + R
        near = np.all((cell >= lo) & (cell <= hi), axis=1)
        outer = np.nonzero(near)[0].astype(np.int64)
        mask = np.zeros(n, dtype=np.uint8)
        mask[elems] = 1
        ptr, ids = candidates(mesh, reach, outer, mask)
        args = _general_args(mesh, space, params, config, outer, ptr, ids,
                             pat, P=PT)
        return int(L.orc_general_core(*args, C.c_void_p(vptr), None))

    nthreads = nthreads or os.cpu_count() or 1
    events = 0
    with ThreadPoolExecutor(max_workers=nthreads) as pool:
        for c in range(1 << dim):
            sel = colour == c
            if not sel.any():
                continue
            ks = key[sel]
            els = inner[sel]
            order = np.argsort(ks, kind="stable")
            ks, els = ks[order], els[order]
            cuts = np.nonzero(np.diff(ks))[0] + 1
            tiles = np.split(els, cuts)
            events += sum(pool.map(run_tile, tiles))
    return events


_PREP_CACHE = {}


def prep_tables_cached(mesh, space, config):
    from paper_2101_08825_b200.assembly import prep_tables
    k = (id(mesh), id(space), repr(config))
    if k not in _PREP_CACHE:
        _PREP_CACHE[k] = prep_tables(mesh, space, config)
    return _PREP_CACHE[k]


def asymmetry_inf(A):
    return float(lib().orc_asymmetry_inf(A.rowptr, A.vals, A.NX, A.NY, A.NZ,
                                         A.K, A.n))


def matvec(A, x):
    y = np.empty(A.n)
    lib().orc_matvec(A.rowptr, A.vals, np.ascontiguousarray(x, np.float64),
                     y, A.NX, A.NY, A.NZ, A.K, A.n)
    return y


def diag(A):
    out = np.empty(A.n)
    lib().orc_diag(A.rowptr, A.vals, A.NX, A.NY, A.K, A.n, out)
    return out


def symmetrize(A):
    lib().orc_symmetrize(A.rowptr, A.vals, A.NX, A.NY, A.NZ, A.K, A.n)


def assemble_general(mesh, space, params, config, census=None):
    """Reference `assemble(..., strategy="general")` + `_finish`, on host.

    Returns a host-only pattern object with vals/events/presym_asymmetry."""
    from paper_2101_08825_b200.assembly import HostPattern
    A = HostPattern.for_space(mesh, space, params, config)
    A.events = run_general(mesh, space, params, config, A, census=census)
    A.vals *= 2.0
    A.presym_asymmetry = asymmetry_inf(A)
    if config.symmetrize:
        symmetrize(A)
    return A
