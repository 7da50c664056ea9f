"""Golden vectors for unstructured Delaunay P1 meshes (BASELINE config #2),
computed by the LIVE reference numba core.

The reference package builds structured meshes only (mesh.py:153-178), but
its pair core `_general_core` (_kernels.py:391-487) is written for
arbitrary affine triangles (`_event_tri`, 146-181) and consumes plain
arrays.  This script builds the Delaunay mesh, FE space, candidate lists
and implicit pattern with the product host layer, then runs the
reference's own `_general_core` on them -- so the fixtures pin the
unstructured path to reference arithmetic, not to a restatement.  Run in
the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \\
        python tests/golden/make_golden_delaunay.py

Stored per case (tests/golden/<name>.npz): meta (json), the mesh arrays the
builder must reproduce (nodes, elem_nodes, elem_cell, elem_color), the
candidate lists, vals (x2 folded), events, asym, rowptr, K.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

# name: (omega, h, delta/h, eps/h, jitter, seed, L_min, L_max, rule)
CASES = {
    "delaunay_tri6": (((0.0, 0.25), (0.0, 0.25)), 1 / 32, 3.0, 0.5, 0.3, 0,
                      1, 3, "tri6"),
    "delaunay_tri7_lmin2": (((0.0, 0.25), (0.0, 0.1875)), 1 / 32, 2.5, 0.25,
                            0.2, 1, 2, 3, "default"),
    "delaunay_eps0": (((0.0, 0.1875), (0.0, 0.1875)), 1 / 32, 2.0, 0.0, 0.3,
                      2, 1, 2, "tri6"),
}


def build(spec):
    sys.path.insert(0, ROOT)
    from paper_2101_08825_b200 import AssemblyConfig, FESpace, KernelParams
    from paper_2101_08825_b200.mesh import build_delaunay_mesh
    omega, h, dr, er, jit, seed, lmin, lmax, rule = spec
    kp = KernelParams(2, dr * h, er * h)
    mesh = build_delaunay_mesh(omega, h, kp.delta + kp.eps, jitter=jit,
                               seed=seed)
    space = FESpace(mesh, 1)
    cfg = AssemblyConfig(L_min=lmin, L_max=lmax, outer_rule=rule,
                         inner_rule=rule, strategy="general")
    return mesh, space, kp, cfg


def run_case(name, spec):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from mollifem import _kernels as RK
    from paper_2101_08825_b200.assembly import HostPattern, prep_tables
    mesh, space, kp, cfg = build(spec)
    n = mesh.n_elements
    outer = np.arange(n, dtype=np.int64)
    ptr, ids = oracle.candidates(mesh, kp.delta + kp.eps, outer,
                                 np.ones(n, np.uint8))
    A = HostPattern.for_space(mesh, space, kp, cfg)
    P = prep_tables(mesh, space, cfg)
    ev = RK._general_core(
        2, 1, mesh.elem_kind, mesh.elem_coords, mesh.elem_lo, mesh.elem_hi,
        space.element_dofs, space.element_nloc, outer, ptr, ids,
        P.box_out_pts, P.box_out_w, P.box_in_pts, P.box_in_w,
        P.tri_out_pts, P.tri_out_w, P.tri_in_pts, P.tri_in_w,
        P.PHI_box_in, P.PHI_tri_in, kp.delta, kp.eps, kp.c_delta_eps,
        cfg.L_min, cfg.L_max, A.gx, A.gy, A.gz, A.NX, A.NY, A.K, A.rowptr,
        A.vals)
    A.vals *= 2.0                                     # _finish
    asym = RK._asymmetry_inf(A.rowptr, A.vals, A.gx, A.gy, A.gz, A.NX, A.NY,
                             A.NZ, A.K, A.n)
    omega, h, dr, er, jit, seed, lmin, lmax, rule = spec
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"),
        meta=json.dumps(dict(name=name, omega=omega, h=h, delta_h=dr,
                             eps_h=er, jitter=jit, seed=seed, L_min=lmin,
                             L_max=lmax, rule=rule)),
        nodes=mesh.nodes, elem_nodes=mesh.elem_nodes,
        elem_cell=mesh.elem_cell, elem_color=mesh.elem_color,
        elem_region=mesh.elem_region, free=space.free,
        cand_ptr=ptr, cand_ids=ids, vals=A.vals, events=np.int64(ev),
        asym=np.float64(asym), rowptr=A.rowptr, K=np.int64(A.K))
    print(f"{name}: n_elem={n} pairs={ptr[-1]} events={ev} nnz={A.nnz} "
          f"colors={mesh.n_colors}", flush=True)


if __name__ == "__main__":
    for k, v in CASES.items():
        if len(sys.argv) == 1 or k in sys.argv[1:]:
            run_case(k, v)
