"""Generate golden vectors from the LIVE reference package.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden.py

For every case in CASES it builds the mesh / FE space / kernel with the
reference package, runs the reference hot path
(assemble(strategy="general") -> _run_general -> _general_core -> _finish,
assembly.py:456-473; _candidates, assembly.py:157-175) and stores inputs and
outputs in tests/golden/<name>.npz:

  meta (json)            case parameters
  elem_*, dofs, free     mesh/FE arrays (pins the host layer)
  cand_ptr, cand_ids     candidate lists over all elements
  vals, events, asym     the assembled matrix (already x2) and diagnostics
  rowptr, K              implicit pattern
  part_*                 a partitioned _run_general (outer subset + inner
                         mask, parallel.py:161-171) when the case asks
  rhs                    assemble_rhs with f=-4 / u=x^2+y^2(+z^2)
                         (harness.py:92-95 manufactured data) when asked

Nothing here runs on the GPU box; the .npz files are the committed fixtures.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# name: (dim, omega, h, delta, eps, kappa, kind, degree, L_min, L_max,
#        outer_rule, inner_rule, extras)
CASES = {
    "tri_p1_lmax3": (2, ((0.0, 0.25), (0.0, 0.25)), 1 / 32, 0.1, 1 / 64, 1.0,
                     "tri", 1, 1, 3, "default", "default", ("rhs", "part")),
    "quad_q1_lmax3": (2, ((0.0, 0.2), (0.0, 0.2)), 0.1, 0.2, 0.05, 1.0,
                      "quad", 1, 1, 3, "default", "default", ("rhs",)),
    "mixed_p1_lmax3": (2, ((0.0, 0.2), (0.0, 0.2)), 0.1, 0.2, 0.05, 1.0,
                       "mixed", 1, 1, 3, "default", "default", ()),
    "quad_q2_lmax2": (2, ((0.0, 0.2), (0.0, 0.2)), 0.1, 0.2, 0.05, 1.0,
                      "quad", 2, 1, 2, "default", "default", ("rhs",)),
    "tri_p2_lmax2": (2, ((0.0, 0.2), (0.0, 0.2)), 0.1, 0.2, 0.05, 1.0,
                     "tri", 2, 1, 2, "default", "default", ()),
    "mixed_q2_lmin2": (2, ((0.0, 0.2), (0.0, 0.3)), 0.1, 0.2, 0.05, 1.0,
                       "mixed", 2, 2, 3, "gauss2", "gauss4", ()),
    "quad_eps0_ties": (2, ((0.0, 0.2), (0.0, 0.2)), 0.1, 0.2, 0.0, 1.0,
                       "quad", 1, 1, 2, "default", "default", ()),
    "quad_lobatto_out": (2, ((0.0, 0.3), (0.0, 0.2)), 0.1, 0.2, 0.05, 1.0,
                         "quad", 1, 1, 3, "lobatto3", "gauss2", ()),
    "tri_p1_deep": (2, ((0.0, 0.1), (0.0, 0.1)), 0.05, 0.1, 0.02, 1.0,
                    "tri", 1, 1, 5, "default", "default", ()),
    "hex_q1_gl3": (3, ((0.0, 0.125),) * 3, 1 / 32, 1.5 / 32, 1 / 64, 2.0,
                   "hex", 1, 1, 2, "default", "default", ("rhs", "part")),
    "hex_q1_gl2_l3": (3, ((0.0, 0.125),) * 3, 1 / 32, 1.5 / 32, 1 / 64, 2.0,
                      "hex", 1, 1, 3, "gauss2", "gauss2", ()),
    "hex_q2_gl3": (3, ((0.0, 0.25),) * 3, 0.125, 0.15, 0.05, 1.0, "hex", 2,
                   1, 2, "default", "default", ()),
}


def run_case(name, spec):
    import mollifem as R
    from mollifem import assembly as RA
    (dim, omega, h, delta, eps, kappa, kind, degree, lmin, lmax, orule,
     irule, extras) = spec
    kp = R.KernelParams(dim, delta, eps, kappa)
    mesh = R.build_mesh(dim, omega, h, delta + eps, kind)
    space = R.FESpace(mesh, degree)
    cfg = R.AssemblyConfig(L_min=lmin, L_max=lmax, outer_rule=orule,
                           inner_rule=irule, strategy="general")
    A = R.assemble(mesh, space, kp, cfg)
    n = mesh.n_elements
    ptr, ids = RA._candidates(mesh, delta + eps, np.arange(n, dtype=np.int64),
                              np.ones(n, dtype=np.bool_))
    out = dict(
        meta=json.dumps(dict(name=name, dim=dim, omega=omega, h=h,
                             delta=delta, eps=eps, kappa=kappa, kind=kind,
                             degree=degree, L_min=lmin, L_max=lmax,
                             outer_rule=orule, inner_rule=irule,
                             extras=list(extras))),
        elem_kind=mesh.elem_kind, elem_proto=mesh.elem_proto,
        elem_region=mesh.elem_region, elem_cell=mesh.elem_cell,
        elem_coords=mesh.elem_coords, elem_lo=mesh.elem_lo,
        elem_hi=mesh.elem_hi, dofs=space.element_dofs,
        nloc=space.element_nloc, free=space.free,
        cand_ptr=ptr, cand_ids=ids, vals=A.vals, events=np.int64(A.events),
        asym=np.float64(A.presym_asymmetry), rowptr=A.rowptr,
        K=np.int64(A.K), c_delta_eps=np.float64(kp.c_delta_eps))
    if kind in ("quad", "tri", "hex"):
        # the reference default strategy ("auto" -> offset-blocked path,
        # assembly.py:448-453, 391-437) on the same problem
        cfg_a = R.AssemblyConfig(L_min=lmin, L_max=lmax, outer_rule=orule,
                                 inner_rule=irule)
        B = R.assemble(mesh, space, kp, cfg_a)
        out.update(vals_auto=B.vals, events_auto=np.int64(B.events),
                   asym_auto=np.float64(B.presym_asymmetry))
    if "part" in extras:
        # one partition of a 2-way RCB split, as parallel_assemble runs it
        from mollifem.parallel import ghost_regions
        pm = R.partition_geometric(mesh, 2)
        regions = ghost_regions(mesh, pm, kp)
        owned = pm.owned(0)
        outer = np.sort(np.concatenate([owned, regions[(1, 0)]]))
        mask = np.zeros(n, dtype=np.bool_)
        mask[owned] = True
        B = A.copy_pattern()
        prep = RA._Prep(mesh, space, kp, cfg)
        ev = RA._run_general(mesh, space, kp, cfg, prep, B,
                             outer_ids=outer.astype(np.int64),
                             inner_mask=mask)
        out.update(part_outer=outer.astype(np.int64), part_owned=owned,
                   part_vals=B.vals, part_events=np.int64(ev),
                   part_owner=pm.owner)
    if "rhs" in extras:
        if dim == 2:
            f = lambda x: np.full(x.shape[:-1], -4.0 * kappa)
            u = lambda x: x[..., 0] ** 2 + x[..., 1] ** 2
        else:
            f = lambda x: np.full(x.shape[:-1], -6.0 * kappa)
            u = lambda x: x[..., 0] ** 2 + x[..., 1] ** 2 + x[..., 2] ** 2
        out["rhs"] = R.assemble_rhs(mesh, space, kp, f, u, A)
        # solver.py:26-90 on the reference matrix ("same solved u" check)
        uh, rep = R.solve(A, out["rhs"], space.free, space.constrained,
                          u(space.dof_coords[space.constrained]))
        out["u"] = uh
        out["u_iters"] = np.int64(rep.iterations)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: n_elem={n} pairs={ptr[-1]} events={A.events} "
          f"nnz={A.nnz}", flush=True)


def main(names=None):
    for name, spec in CASES.items():
        if names and name not in names:
            continue
        run_case(name, spec)


if __name__ == "__main__":
    main(sys.argv[1:])
