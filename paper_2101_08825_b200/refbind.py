"""Reference-side bindings: the B200 library behind the reference's own hooks.

The reference package (`mollifem`) runs its hot path through two
functions:

  _general_core(...)   _kernels.py:391-487, called by _run_general with
                       plain numpy arrays and explicit candidate lists;
  _run_general(...)    assembly.py:369-388, which builds the lists
                       (`_candidates`) and calls _general_core.

This module provides both with the reference's exact signatures, taking the
reference's own objects (its `Mesh`, `FESpace`, `_Prep`, `SparseMatrix`) or
arrays, and accumulating into the caller's host `vals` like the numba cores
do.  A maintainer binds the reference to the B200 path with

    import mollifem.assembly, mollifem._kernels
    from paper_2101_08825_b200 import refbind
    mollifem.assembly._run_general = refbind.run_general      # fast path
    # or, at the array level:
    mollifem._kernels._general_core = refbind.general_core

(INTEGRATION.md section 2).  `run_general` sends the pair set it is given
(outer ids x inner mask, gap < delta+eps) to `mf_general_core`, which runs
the specialised kernels; `general_core` sends explicit lists to
`mf_general_core_lists` (every listed pair, the generic kernel).  Both need
a CUDA device and fail loudly without one.
"""

import ctypes

import numpy as np

from . import _native as N

__all__ = ["run_general", "general_core"]


def _box_1d(mesh, config):
    """1D factors of the tensor box rules for the sum-factorised kernels
    (None when the preset is not a tensor Gauss/Lobatto rule)."""
    from .assembly import rule_1d
    if mesh.dim not in (2, 3) or getattr(mesh, "kind", "") not in (
            "quad", "hex", "mixed"):
        return None
    try:
        return rule_1d(config.outer_rule), rule_1d(config.inner_rule)
    except ValueError:
        return None


def run_general(mesh, space, params, config, prep, A, outer_ids=None,
                inner_mask=None, device=None):
    """`_run_general` (assembly.py:369-388) on the B200: every pair (l, m)
    with l in outer_ids, inner_mask[m] and box gap < delta+eps; adds the
    blocks (unscaled, like the reference) into the host `A.vals` and
    returns the event count."""
    import torch
    from .assembly import stencil_radius
    from .device import ColorPlan, DeviceMesh, DeviceRules, to_device
    n = mesh.n_elements
    outer = (np.arange(n, dtype=np.int64) if outer_ids is None
             else np.ascontiguousarray(outer_ids, dtype=np.int64))
    if outer.size and (outer.min() < 0 or outer.max() >= n):
        raise ValueError("outer id out of range")
    if outer.size != np.unique(outer).size:
        # repeated outer ids repeat their pairs in the reference: take the
        # explicit-list path, which honours every listed pair
        return _run_general_lists(mesh, space, params, config, prep, A,
                                  outer, inner_mask, device)
    mask = (np.ones(n, dtype=bool) if inner_mask is None
            else np.asarray(inner_mask).astype(bool))
    dmesh = DeviceMesh(mesh, space, device)
    dev = dmesh.device
    drules = DeviceRules(prep, dev, box_1d=_box_1d(mesh, config))
    om = np.zeros(n, dtype=np.uint8)
    om[outer] = 1
    om_d = to_device(om, dev)
    plan = ColorPlan(mesh, np.nonzero(mask)[0], dev)
    rowptr = to_device(np.ascontiguousarray(A.rowptr, np.int64), dev)
    pat = N.MfPattern(NX=A.NX, NY=A.NY, NZ=A.NZ, K=A.K, n=A.n,
                      rowptr=rowptr.data_ptr())
    kern = N.MfKernel(delta=params.delta, eps=params.eps,
                      cde=params.c_delta_eps, L_min=config.L_min,
                      L_max=config.L_max)
    vals = torch.zeros(int(A.rowptr[-1]), dtype=torch.float64, device=dev)
    cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=dev)
    L = N.lib()
    wsb = int(L.mf_general_workspace_bytes(ctypes.byref(dmesh.struct),
                                           ctypes.byref(drules.struct),
                                           plan.n_inner))
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device=dev)
    cptr = np.ascontiguousarray(plan.color_ptr)
    R = stencil_radius(params.delta + params.eps, mesh.h)
    with torch.cuda.device(dev):
        N.check(L.mf_general_core(
            ctypes.byref(dmesh.struct), ctypes.byref(drules.struct),
            ctypes.byref(kern), ctypes.byref(pat), N.ptr(om_d),
            N.ptr(plan.inner_sorted), cptr.ctypes.data_as(ctypes.c_void_p),
            plan.ngroups, R, 1.0, N.ptr(vals), N.ptr(cnt), 0, N.ptr(ws), wsb,
            N.stream_ptr(torch.cuda.current_stream(dev))), "mf_general_core")
        return _finish_host(A, vals, cnt)


def _finish_host(A, vals, cnt):
    from .assembly import check_counters
    c = cnt.cpu().numpy()
    check_counters(c)
    A.vals += vals.cpu().numpy()
    return int(c[N.CNT_EVENTS])


def _run_general_lists(mesh, space, params, config, prep, A, outer,
                       inner_mask, device):
    from .assembly import candidates
    n = mesh.n_elements
    mask = (np.ones(n, dtype=np.uint8) if inner_mask is None
            else np.asarray(inner_mask).astype(np.uint8))
    ptr, ids = candidates(mesh, params.delta + params.eps, outer, mask,
                          device=device)
    return general_core(
        mesh.dim, space.degree, mesh.elem_kind, mesh.elem_coords,
        mesh.elem_lo, mesh.elem_hi, space.element_dofs,
        getattr(space, "element_nloc", None), outer, ptr, ids,
        prep.box_out_pts, prep.box_out_w, prep.box_in_pts, prep.box_in_w,
        prep.tri_out_pts, prep.tri_out_w, prep.tri_in_pts, prep.tri_in_w,
        prep.PHI_box_in, prep.PHI_tri_in, params.delta, params.eps,
        params.c_delta_eps, config.L_min, config.L_max, A.gx, A.gy, A.gz,
        A.NX, A.NY, A.K, A.rowptr, A.vals, device=device)


def general_core(dim, degree, elem_kind, elem_coords, elem_lo, elem_hi,
                 elem_dofs, elem_nloc, outer_ids, cand_ptr, cand_ids,
                 box_out_pts, box_out_w, box_in_pts, box_in_w,
                 tri_out_pts, tri_out_w, tri_in_pts, tri_in_w,
                 PHI1_box, PHI1_tri, delta, eps, cde, L_min, L_max,
                 gx, gy, gz, NX, NY, K, rowptr, vals, device=None):
    """`_general_core` (_kernels.py:391-400) with its exact arguments: runs
    every listed pair (outer_ids[i], cand_ids[k]) on the B200 and adds the
    blocks into the host array `vals` in place; returns the event count.
    elem_nloc is accepted for signature parity (the kernels take nloc from
    the element kind and degree, as the reference's element_nloc does)."""
    import torch
    from .device import _dev, to_device
    dev = _dev(device)
    if not 1 <= L_min <= L_max or L_max > 24:
        raise ValueError("need 1 <= L_min <= L_max <= 24")
    kind = np.ascontiguousarray(elem_kind, np.int8)
    coords = np.ascontiguousarray(elem_coords, np.float64)
    dofs = np.ascontiguousarray(elem_dofs, np.int64)
    n = int(kind.shape[0])
    keep = []

    def d(a, dt=np.float64):
        t = to_device(np.ascontiguousarray(a, dt), dev)
        keep.append(t)
        return t.data_ptr()

    kinds = np.unique(kind).astype(np.int64) if n else np.zeros(0, np.int64)
    mesh = N.MfMesh(
        dim=int(dim), degree=int(degree), n_elem=n,
        nv_max=int(coords.shape[1]), nloc_max=int(dofs.shape[1]),
        elem_kind=d(kind, np.int8), elem_coords=d(coords),
        elem_lo=d(elem_lo), elem_hi=d(elem_hi), elem_dofs=d(dofs, np.int64),
        elem_cell=None, cell_ptr=None, ncx=1, ncy=1, ncz=1,
        kinds_present=int(np.bitwise_or.reduce(1 << kinds)) if n else 0,
        layout=0, row_period=2)
    rules = N.MfRules(
        nq_box_out=len(box_out_w), nq_box_in=len(box_in_w),
        nq_tri_out=len(tri_out_w), nq_tri_in=len(tri_in_w),
        box_out_pts=d(box_out_pts), box_out_w=d(box_out_w),
        box_in_pts=d(box_in_pts), box_in_w=d(box_in_w),
        tri_out_pts=d(tri_out_pts), tri_out_w=d(tri_out_w),
        tri_in_pts=d(tri_in_pts), tri_in_w=d(tri_in_w),
        phi_box_in=d(PHI1_box), phi_tri_in=d(PHI1_tri),
        n1d_box_out=0, n1d_box_in=0, box_out_x1d=None, box_out_w1d=None,
        box_in_x1d=None, box_in_w1d=None)
    kern = N.MfKernel(delta=float(delta), eps=float(eps), cde=float(cde),
                      L_min=int(L_min), L_max=int(L_max))
    rp = np.ascontiguousarray(rowptr, np.int64)
    nrows = rp.shape[0] - 1
    NZ = nrows // (int(NX) * int(NY)) if nrows else 1
    pat = N.MfPattern(NX=int(NX), NY=int(NY), NZ=max(NZ, 1), K=int(K),
                      n=nrows, rowptr=d(rp, np.int64))
    outer = np.ascontiguousarray(outer_ids, np.int64)
    out_d = to_device(outer if outer.size else np.zeros(1, np.int64), dev)
    ptr_d = to_device(np.ascontiguousarray(cand_ptr, np.int64), dev)
    ids = np.ascontiguousarray(cand_ids, np.int64)
    ids_d = to_device(ids if ids.size else np.zeros(1, np.int64), dev)
    out = torch.zeros(int(rp[-1]) if nrows else 0, dtype=torch.float64,
                      device=dev)
    cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        N.check(N.lib().mf_general_core_lists(
            ctypes.byref(mesh), ctypes.byref(rules), ctypes.byref(kern),
            ctypes.byref(pat), N.ptr(out_d), int(outer.size), N.ptr(ptr_d),
            N.ptr(ids_d), 1.0, N.ptr(out), N.ptr(cnt), 0,
            N.stream_ptr(torch.cuda.current_stream(dev))),
            "mf_general_core_lists")
        from .assembly import check_counters
        c = cnt.cpu().numpy()
        check_counters(c)
        vals += out.cpu().numpy()
    return int(c[N.CNT_EVENTS])
