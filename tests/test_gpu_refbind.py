"""The reference-side binding on the GPU.

`refbind.run_general` / `refbind.general_core` replace the reference's
`_run_general` (assembly.py:369-388) and `_general_core`
(_kernels.py:391-487).  Here they are driven exactly as the reference
drives them -- with objects that carry ONLY the reference's attributes
(its Mesh, FESpace, _Prep, SparseMatrix; none of our host-layer methods
such as `cell_ptr()` or the 1D rule factors) and with the argument list
_run_general passes to _general_core -- and the result is compared with
the live-reference golden fixtures.
"""

import types

import numpy as np
import pytest

from conftest import Golden, rel_frob

pytestmark = pytest.mark.gpu

CASES = ["tri_p1_lmax3", "hex_q1_gl3", "mixed_p1_lmax3", "quad_q2_lmax2",
         "hex_q2_gl3", "quad_eps0_ties"]


def _reference_shaped(mesh, space, kp, cfg):
    """Stand-ins with exactly the reference's attribute sets
    (mesh.py:75-122, fe_space.py:83-164, assembly.py:189-223, 333-356)."""
    from paper_2101_08825_b200.assembly import HostPattern, pattern_halfwidth
    from paper_2101_08825_b200.assembly import prep_tables
    m = types.SimpleNamespace(
        dim=mesh.dim, h=mesh.h, kind=mesh.kind,
        grid_ncells=np.asarray(mesh.grid_ncells),
        n_elements=mesh.n_elements, elem_kind=mesh.elem_kind,
        elem_proto=mesh.elem_proto, elem_region=mesh.elem_region,
        elem_cell=mesh.elem_cell, elem_coords=mesh.elem_coords,
        elem_lo=mesh.elem_lo, elem_hi=mesh.elem_hi)
    s = types.SimpleNamespace(degree=space.degree,
                              element_dofs=space.element_dofs,
                              element_nloc=space.element_nloc,
                              n_dofs=space.n_dofs)
    P = prep_tables(mesh, space, cfg)
    names = ["box_out_pts", "box_out_w", "box_in_pts", "box_in_w",
             "tri_out_pts", "tri_out_w", "tri_in_pts", "tri_in_w",
             "PHI_box_in", "PHI_tri_in"]
    prep = types.SimpleNamespace(**{k: getattr(P, k) for k in names})
    K, _ = pattern_halfwidth(mesh, kp, cfg, space.degree)
    H = HostPattern(space, K)
    A = types.SimpleNamespace(NX=H.NX, NY=H.NY, NZ=H.NZ, K=H.K, n=H.n,
                              gx=H.gx, gy=H.gy, gz=H.gz, rowptr=H.rowptr,
                              vals=np.zeros(H.nnz))
    return m, s, prep, A


@pytest.mark.parametrize("name", CASES)
def test_run_general_binding_matches_reference(name):
    from paper_2101_08825_b200 import refbind
    g = Golden(name)
    mesh, space, kp, cfg = g.build()
    m, s, prep, A = _reference_shaped(mesh, space, kp, cfg)
    ev = refbind.run_general(m, s, kp, cfg, prep, A)
    A.vals *= 2.0                      # _finish (assembly.py:440-445)
    assert ev == int(g["events"])
    assert rel_frob(A.vals, g["vals"]) <= 1e-10


@pytest.mark.parametrize("name", CASES)
def test_general_core_binding_matches_reference(name):
    """The array-level hook with the argument list of assembly.py:378-386
    and the reference's candidate lists."""
    import oracle
    from paper_2101_08825_b200 import refbind
    g = Golden(name)
    mesh, space, kp, cfg = g.build()
    m, s, prep, A = _reference_shaped(mesh, space, kp, cfg)
    n = mesh.n_elements
    outer = np.arange(n, dtype=np.int64)
    ptr, ids = oracle.candidates(mesh, kp.delta + kp.eps, outer,
                                 np.ones(n, np.uint8))
    ev = refbind.general_core(
        m.dim, s.degree, m.elem_kind, m.elem_coords, m.elem_lo, m.elem_hi,
        s.element_dofs, s.element_nloc, outer, ptr, ids,
        prep.box_out_pts, prep.box_out_w, prep.box_in_pts, prep.box_in_w,
        prep.tri_out_pts, prep.tri_out_w, prep.tri_in_pts, prep.tri_in_w,
        prep.PHI_box_in, prep.PHI_tri_in, kp.delta, kp.eps, kp.c_delta_eps,
        cfg.L_min, cfg.L_max, A.gx, A.gy, A.gz, A.NX, A.NY, A.K, A.rowptr,
        A.vals)
    A.vals *= 2.0
    assert ev == int(g["events"])
    assert rel_frob(A.vals, g["vals"]) <= 1e-10


def test_general_core_lists_partition_and_duplicates():
    """Lists that are not a product set: a partition golden
    (outer = owned + ghosts, inner = owned) and a list with a repeated
    pair, which the reference counts twice."""
    import oracle
    from paper_2101_08825_b200 import refbind
    from paper_2101_08825_b200.assembly import HostPattern
    g = Golden("hex_q1_gl3")
    mesh, space, kp, cfg = g.build()
    m, s, prep, A = _reference_shaped(mesh, space, kp, cfg)
    n = mesh.n_elements
    rng = np.random.default_rng(3)
    outer = np.sort(rng.choice(n, n // 3, replace=False)).astype(np.int64)
    mask = (rng.random(n) < 0.5).astype(np.uint8)
    ptr, ids = oracle.candidates(mesh, kp.delta + kp.eps, outer, mask)
    # repeat the first list entry once (outer 0's first candidate twice)
    ids2 = np.insert(ids, 0, ids[0])
    ptr2 = ptr.copy()
    ptr2[1:] += 1

    def run(p, i):
        B = HostPattern(space, A.K)
        ev = refbind.general_core(
            m.dim, s.degree, m.elem_kind, m.elem_coords, m.elem_lo,
            m.elem_hi, s.element_dofs, s.element_nloc, outer, p, i,
            prep.box_out_pts, prep.box_out_w, prep.box_in_pts,
            prep.box_in_w, prep.tri_out_pts, prep.tri_out_w,
            prep.tri_in_pts, prep.tri_in_w, prep.PHI_box_in,
            prep.PHI_tri_in, kp.delta, kp.eps, kp.c_delta_eps, cfg.L_min,
            cfg.L_max, A.gx, A.gy, A.gz, A.NX, A.NY, A.K, A.rowptr, B.vals)
        return ev, B.vals

    R = HostPattern(space, A.K)
    ev_o = oracle.run_general(mesh, space, kp, cfg, R, outer_ids=outer,
                              inner_mask=mask)
    ev, v = run(ptr, ids)
    assert ev == ev_o and rel_frob(v, R.vals) <= 1e-10
    R2 = HostPattern(space, A.K)
    one = np.zeros(n, np.uint8)
    one[ids[0]] = 1
    ev_one = oracle.run_general(mesh, space, kp, cfg, R2,
                                outer_ids=outer[:1], inner_mask=one)
    ev2, v2 = run(ptr2, ids2)
    assert ev2 == ev_o + ev_one
    assert rel_frob(v2, R.vals + R2.vals) <= 1e-10


def test_general_core_lists_rejects_bad_ids():
    import oracle
    from paper_2101_08825_b200 import refbind
    g = Golden("tri_p1_lmax3")
    mesh, space, kp, cfg = g.build()
    m, s, prep, A = _reference_shaped(mesh, space, kp, cfg)
    n = mesh.n_elements
    outer = np.arange(4, dtype=np.int64)
    ptr, ids = oracle.candidates(mesh, kp.delta + kp.eps, outer,
                                 np.ones(n, np.uint8))
    bad = ids.copy()
    bad[-1] = n + 5

    def call(o, i):
        return refbind.general_core(
            m.dim, s.degree, m.elem_kind, m.elem_coords, m.elem_lo,
            m.elem_hi, s.element_dofs, s.element_nloc, o, ptr, i,
            prep.box_out_pts, prep.box_out_w, prep.box_in_pts,
            prep.box_in_w, prep.tri_out_pts, prep.tri_out_w,
            prep.tri_in_pts, prep.tri_in_w, prep.PHI_box_in,
            prep.PHI_tri_in, kp.delta, kp.eps, kp.c_delta_eps, cfg.L_min,
            cfg.L_max, A.gx, A.gy, A.gz, A.NX, A.NY, A.K, A.rowptr, A.vals)

    with pytest.raises(RuntimeError, match="out of range"):
        call(outer, bad)
    with pytest.raises(RuntimeError, match="out of range"):
        call(np.array([0, 1, 2, n], np.int64), ids)
    assert float(np.abs(A.vals).max()) == 0.0


@pytest.mark.parametrize("name", ["hex_q1_gl3", "tri_p1_lmax3"])
def test_unmodified_reference_package_bound_to_b200(name, monkeypatch):
    """The reference package itself (installed under baseline/_ref) with
    its hooks bound to the B200 library, as INTEGRATION.md section 2 shows:
    its own assemble() and parallel_assemble() then match its golden
    outputs."""
    import bench
    mf = bench.ref_import()
    if mf is None:
        pytest.skip("reference not installed under baseline/_ref")
    from mollifem import _kernels as RK
    from mollifem import assembly as RA
    from mollifem import parallel as RP
    from paper_2101_08825_b200 import refbind
    g = Golden(name)
    m = g.meta
    mesh = mf.build_mesh(m["dim"], m["omega"], m["h"], m["delta"] + m["eps"],
                         m["kind"])
    space = mf.FESpace(mesh, m["degree"])
    kp = mf.KernelParams(m["dim"], m["delta"], m["eps"], m["kappa"])
    cfg = mf.AssemblyConfig(L_min=m["L_min"], L_max=m["L_max"],
                            outer_rule=m["outer_rule"],
                            inner_rule=m["inner_rule"], strategy="general")
    monkeypatch.setattr(RA, "_run_general", refbind.run_general)
    monkeypatch.setattr(RP, "_run_general", refbind.run_general)
    A = mf.assemble(mesh, space, kp, cfg)
    assert A.events == int(g["events"])
    assert rel_frob(A.vals, g["vals"]) <= 1e-10
    B, ctxs = mf.parallel_assemble(mesh, space, kp, cfg, n_parts=3)
    assert B.events == int(g["events"])
    assert rel_frob(B.vals, g["vals"]) <= 1e-10
    # one level lower: the array-level core
    monkeypatch.undo()
    monkeypatch.setattr(RK, "_general_core", refbind.general_core)
    C = mf.assemble(mesh, space, kp, cfg)
    assert C.events == int(g["events"])
    assert rel_frob(C.vals, g["vals"]) <= 1e-10
