"""Tetrahedral P1 elements (BASELINE configs #4/#5 as written; SURVEY.md
8(f) f2).

The reference has no tetrahedra, so parity for this
element is unpinned against it.  The checks are instead:
  * the quadrature rules integrate monomials exactly to their degree;
  * the 6-tet Kuhn mesh (with and without jitter) tiles the box
    conformingly with positively oriented tets, and the FE space numbers
    the vertices as DOFs;
  * the C restatement (oracle/mf_oracle.c event_tet / tet_children) obeys
    the identities the reference tests for its own elements: A 1 = 0
    (test_assembly.py:49-55), partition invariance (test_parallel.py:
    93-114), and the blocks reduce to the known constant-kernel values;
  * the GPU kernel (mf_tet.cu, through the C-ABI) matches the oracle with
    identical event counts and matrices within 1e-10 relative Frobenius
    norm, with and without jitter, eps > 0 and eps = 0, for 1/4/11-point
    rules and L_max 2..3.
"""

import itertools
import math

import numpy as np
import pytest

from conftest import rel_frob

TOL = 1e-10

# name: (omega side, h, delta, eps, jitter, outer, inner, L_min, L_max)
CASES = {
    "tet4_l2": (0.125, 1 / 16, 0.08, 1 / 32, 0.0, "default", "default", 1,
                2),
    "tet4_l3_jit": (0.125, 1 / 16, 0.08, 1 / 32, 0.1, "default", "default",
                    1, 3),
    "tet11_l2_jit": (0.125, 1 / 16, 0.08, 1 / 64, 0.1, "tet11", "tet11", 1,
                     2),
    "tet4_eps0": (0.125, 1 / 16, 0.08, 0.0, 0.0, "default", "default", 1, 2),
    "tet1_lmin2": (0.125, 1 / 16, 0.08, 1 / 32, 0.05, "tet1", "tet4", 2, 3),
    "wide_tet1": (0.0625, 1 / 16, 0.1875, 1 / 32, 0.1, "tet1", "tet1", 1, 2),
}


def build(name):
    from paper_2101_08825_b200 import (AssemblyConfig, FESpace, KernelParams,
                                       build_mesh)
    side, h, d, e, jit, orr, irr, lmin, lmax = CASES[name]
    mesh = build_mesh(3, ((0.0, side),) * 3, h, d + e, "tet", jitter=jit,
                      seed=7)
    space = FESpace(mesh, 1)
    kp = KernelParams(3, d, e, 2.0)
    cfg = AssemblyConfig(L_min=lmin, L_max=lmax, outer_rule=orr,
                         inner_rule=irr, strategy="general")
    return mesh, space, kp, cfg


_ORACLE = {}


def oracle_matrix(name):
    if name not in _ORACLE:
        import oracle
        oracle.build()
        mesh, space, kp, cfg = build(name)
        _ORACLE[name] = oracle.assemble_general(mesh, space, kp, cfg)
    return _ORACLE[name]


# ---------------------------------------------------------------- host/CPU

@pytest.mark.parametrize("n", [1, 4, 11])
def test_tet_rule_exactness(n):
    from paper_2101_08825_b200.quadrature import tet_rule
    r = tet_rule(n)
    P, W = r.ref_points, r.weights
    assert abs(W.sum() - 1.0 / 6.0) < 1e-15
    for a, b, c in itertools.product(range(r.exact_degree + 1), repeat=3):
        if a + b + c > r.exact_degree:
            continue
        exact = (math.factorial(a) * math.factorial(b) * math.factorial(c)
                 / math.factorial(a + b + c + 3))
        q = float((W * P[:, 0] ** a * P[:, 1] ** b * P[:, 2] ** c).sum())
        assert abs(q - exact) < 1e-15, (n, a, b, c)
    # one degree higher is not exact for at least one monomial
    worst = max(abs(float((W * P[:, 0] ** a * P[:, 1] ** b
                           * P[:, 2] ** c).sum())
                    - math.factorial(a) * math.factorial(b)
                    * math.factorial(c) / math.factorial(a + b + c + 3))
                for a, b, c in itertools.product(range(r.exact_degree + 2),
                                                 repeat=3)
                if a + b + c == r.exact_degree + 1)
    assert worst > 1e-12


def test_tet_presets():
    from paper_2101_08825_b200.quadrature import rule_for_kind
    assert len(rule_for_kind("tet").weights) == 4
    assert len(rule_for_kind("tet", "tet11").weights) == 11
    with pytest.raises(ValueError):
        rule_for_kind("hex", "tet4")


@pytest.mark.parametrize("jitter", [0.0, 0.1])
def test_tet_mesh_conforming(jitter):
    from paper_2101_08825_b200 import build_mesh
    mesh = build_mesh(3, ((0.0, 0.25),) * 3, 1 / 16, 0.1, "tet",
                      jitter=jitter, seed=5)
    c = mesh.elem_coords
    det = np.linalg.det(np.stack([c[:, 1] - c[:, 0], c[:, 2] - c[:, 0],
                                  c[:, 3] - c[:, 0]], axis=2))
    assert (det > 0.3 * mesh.h ** 3).all()
    box = np.asarray(mesh.grid_ncells) * mesh.h
    assert abs(det.sum() / 6.0 - box.prod()) < 1e-12
    # every interior face is shared by exactly two tets, boundary faces by
    # one, and boundary faces lie on the outer box
    faces = {}
    for e, nodes in enumerate(mesh.elem_nodes):
        for f in itertools.combinations(sorted(nodes.tolist()), 3):
            faces.setdefault(f, []).append(e)
    counts = np.array([len(v) for v in faces.values()])
    assert set(counts.tolist()) <= {1, 2}
    lo = np.asarray(mesh.grid_origin)
    hi = lo + box
    for f, owners in faces.items():
        if len(owners) == 1:
            p = mesh.nodes[list(f)]
            on = np.isclose(p, lo).all(axis=0) | np.isclose(p, hi).all(axis=0)
            assert on.any()
    # elements are cell-lex ordered, 6 protos per cell
    assert (mesh.elem_proto == np.tile(np.arange(6), len(c) // 6)).all()
    assert (np.diff(mesh.cell_flat()) >= 0).all()


def test_tet_jitter_keeps_regions():
    from paper_2101_08825_b200 import FESpace, build_mesh
    m0 = build_mesh(3, ((0.0, 0.25),) * 3, 1 / 16, 0.1, "tet")
    m1 = build_mesh(3, ((0.0, 0.25),) * 3, 1 / 16, 0.1, "tet", jitter=0.1,
                    seed=1)
    d = np.abs(m1.nodes - m0.nodes)
    assert d.max() <= 0.1 * m0.h + 1e-15 and d.max() > 0.05 * m0.h
    # Omega elements stay inside Omega, Gamma elements outside
    om = m1.elem_region == 0
    assert (m1.elem_lo[om] >= -1e-15).all() and (m1.elem_hi[om] <= 0.25
                                                  + 1e-15).all()
    s = FESpace(m1, 1)
    assert np.array_equal(s.element_dofs, m1.elem_nodes)
    assert np.array_equal(s.dof_coords, m1.nodes)
    s0 = FESpace(m0, 1)
    assert np.array_equal(s.free, s0.free)
    assert m1.stencil_pad == pytest.approx(0.2 / 16)
    with pytest.raises(ValueError):
        FESpace(m1, 2)
    with pytest.raises(ValueError):
        build_mesh(3, ((0.0, 0.25),) * 3, 1 / 16, 0.1, "hex", jitter=0.1)


def test_tet_candidates_cover_jitter():
    """The padded stencil finds every pair a brute-force box test finds."""
    import oracle
    oracle.build()
    from paper_2101_08825_b200 import build_mesh
    mesh = build_mesh(3, ((0.0, 0.125),) * 3, 1 / 16, 0.11, "tet",
                      jitter=0.2, seed=3)
    n = mesh.n_elements
    ptr, ids = oracle.candidates(mesh, 0.11, np.arange(n),
                                 np.ones(n, np.uint8))
    lo, hi = mesh.elem_lo, mesh.elem_hi
    for l in range(0, n, 97):
        gap = np.maximum(np.maximum(lo - hi[l], lo[l] - hi), 0.0).max(axis=1)
        want = np.nonzero(gap < 0.11)[0]
        assert np.array_equal(ids[ptr[l]:ptr[l + 1]], want)


def test_tet_oracle_identities():
    """A 1 = 0, near-symmetry and partition invariance on the oracle."""
    import oracle
    from paper_2101_08825_b200.assembly import HostPattern
    mesh, space, kp, cfg = build("tet4_l3_jit")
    A = oracle_matrix("tet4_l3_jit")
    assert np.abs(oracle.matvec(A, np.ones(A.n))).max() < 1e-13 * np.abs(
        A.vals).max()
    assert A.presym_asymmetry < 0.05 * np.abs(A.vals).max()
    # two inner-element halves with all outer elements: same matrix
    n = mesh.n_elements
    B = HostPattern.for_space(mesh, space, kp, cfg)
    ev = 0
    for half in (np.arange(n) < n // 2, np.arange(n) >= n // 2):
        ev += oracle.run_general(mesh, space, kp, cfg, B,
                                 inner_mask=half.astype(np.uint8))
    B.vals *= 2.0
    assert ev == A.events
    assert rel_frob(B.vals, A.vals) < 1e-14


def test_tet_oracle_linear_patch():
    """For u linear, (A u)_i = 0 on rows whose whole delta+eps neighbourhood
    is inside the mesh: the nonlocal operator of a linear field vanishes
    up to the quadrature error of the mollified kernel (symmetric ball),
    which shrinks with L_max."""
    import oracle
    mesh, space, kp, cfg = build("tet4_l2")
    A = oracle_matrix("tet4_l2")
    u = space.dof_coords @ np.array([1.0, -2.0, 0.5])
    r = oracle.matvec(A, u)
    c = space.dof_coords
    reach = kp.delta + kp.eps + mesh.h - 1e-9
    lo = np.asarray(mesh.grid_origin)
    hi = lo + np.asarray(mesh.grid_ncells) * mesh.h
    inner = ((c - lo > reach) & (hi - c > reach)).all(axis=1)
    assert inner.any()
    scale = np.abs(A.vals).max() * np.abs(u).max()
    assert np.abs(r[inner]).max() < 1e-6 * scale
    assert np.abs(r).max() > 1e-3 * scale      # boundary rows do not vanish


# ---------------------------------------------------------------- GPU

def test_bey_corner_child_box_from_root_box():
    """k_tet's batched leaf classification (mf_tet.cu, ST_RBOX) takes the
    vertex box of corner child b of Bey's refinement as mid(v_b, root box)
    instead of the min/max over the child's 4 vertices.  Rounding is
    monotone, so the two are the same bits: checked here on random,
    jitter-like and degenerate-tie coordinates."""
    rng = np.random.default_rng(7)
    for trial in range(2000):
        if trial % 3 == 0:       # lattice + jitter, many equal coordinates
            v = (rng.integers(0, 3, (4, 3)) / 64.0
                 + (trial % 2) * rng.uniform(-0.1, 0.1, (4, 3)) / 64.0 + 0.3)
        elif trial % 3 == 1:     # wide dynamic range, both signs
            v = rng.standard_normal((4, 3)) * 10.0 ** rng.integers(-8, 8)
        else:
            v = rng.uniform(-1.0, 2.0, (4, 3))
        lo, hi = v.min(axis=0), v.max(axis=0)
        for b in range(4):
            child = np.array([v[b] if j == b else 0.5 * (v[b] + v[j])
                              for j in range(4)])
            assert np.array_equal(child.min(axis=0), 0.5 * (v[b] + lo))
            assert np.array_equal(child.max(axis=0), 0.5 * (v[b] + hi))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_tet_gpu_matches_oracle(name):
    from paper_2101_08825_b200 import assemble
    mesh, space, kp, cfg = build(name)
    A = assemble(mesh, space, kp, cfg)
    R = oracle_matrix(name)
    assert np.array_equal(A.rowptr, R.rowptr) and A.K == R.K
    assert A.events == R.events
    err = rel_frob(A.vals, R.vals)
    print(f"{name}: events={A.events} relF={err:.3e}")
    assert err <= TOL
    assert abs(A.presym_asymmetry - R.presym_asymmetry) <= 1e-9 * np.abs(
        R.vals).max()


@pytest.mark.gpu
def test_tet_gpu_noshortcuts_and_auto():
    from paper_2101_08825_b200 import AssemblyConfig, assemble
    mesh, space, kp, cfg = build("tet4_l2")
    R = oracle_matrix("tet4_l2")
    A = assemble(mesh, space, kp, cfg, flags=2)       # every event full
    assert A.events == R.events and rel_frob(A.vals, R.vals) <= TOL
    auto = AssemblyConfig(L_max=cfg.L_max)            # "auto" -> general
    B = assemble(mesh, space, kp, auto)
    assert B.events == R.events and rel_frob(B.vals, R.vals) <= TOL
    with pytest.raises(ValueError):
        assemble(mesh, space, kp, AssemblyConfig(L_max=2,
                                                 strategy="blocked"))


@pytest.mark.gpu
def test_tet_gpu_rhs_and_solve():
    """Load vector against a host numpy restatement, then the GPU solve of
    the manufactured problem against a CPU solve of the oracle matrix."""
    import scipy.sparse.linalg as spla
    from paper_2101_08825_b200 import assemble, assemble_rhs, solve
    from paper_2101_08825_b200.quadrature import tet_rule
    mesh, space, kp, cfg = build("tet4_l3_jit")
    A = assemble(mesh, space, kp, cfg)
    f = lambda x: -12.0 + 0.0 * x[..., 0]          # kappa = 2: -2*kappa*3
    g = lambda x: (x ** 2).sum(axis=-1)
    rhs = assemble_rhs(mesh, space, kp, f, g, A)
    # host restatement of the load: tet11 on Omega elements
    r = tet_rule(11)
    load = np.zeros(space.n_dofs)
    for e in mesh.omega_element_ids():
        v = mesh.elem_coords[e]
        E = np.column_stack([v[1] - v[0], v[2] - v[0], v[3] - v[0]])
        det = abs(np.linalg.det(E))
        pts = v[0] + r.ref_points @ E.T
        lam = np.column_stack([1 - r.ref_points.sum(axis=1), r.ref_points])
        load[space.element_dofs[e]] += det * (r.weights * f(pts)) @ lam
    gt = np.zeros(space.n_dofs)
    gt[space.constrained] = g(space.dof_coords[space.constrained])
    R = oracle_matrix("tet4_l3_jit")
    import oracle
    want = (load - oracle.matvec(R, gt))[space.free]
    assert np.abs(rhs - want).max() <= 1e-9 * np.abs(want).max()
    u, rep = solve(A, rhs, space.free, space.constrained,
                   g(space.dof_coords[space.constrained]))
    assert rep.converged
    S = A.to_scipy()                 # same pattern, oracle values
    S.data = R.vals.copy()
    Aff = S[space.free][:, space.free]
    ref = spla.spsolve(Aff.tocsc(), want)
    assert np.abs(u[space.free] - ref).max() <= 1e-8 * max(
        1.0, np.abs(ref).max())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tet4_l3_jit", "tet11_l2_jit"])
def test_tet_gpu_partitions_and_slabs(name):
    """Partition invariance (parallel_assemble, RCB + ghost regions) and the
    z-slab decomposition of the multi-GPU path, emulated on one device."""
    from paper_2101_08825_b200.parallel import emulate_slabs, parallel_assemble
    mesh, space, kp, cfg = build(name)
    R = oracle_matrix(name)
    for n_parts in (2, 3):
        A, ctxs = parallel_assemble(mesh, space, kp, cfg, n_parts=n_parts)
        assert A.events == R.events
        assert rel_frob(A.vals, R.vals) <= 1e-12
    for world in (2, 3):
        full, events = emulate_slabs(mesh, space, kp, cfg, world)
        assert events == R.events
        assert rel_frob(full.cpu().numpy(), R.vals) <= 1e-12


@pytest.mark.gpu
def test_tet_gpu_deterministic():
    from paper_2101_08825_b200 import assemble
    mesh, space, kp, cfg = build("tet4_l3_jit")
    a = assemble(mesh, space, kp, cfg).vals
    b = assemble(mesh, space, kp, cfg).vals
    assert np.array_equal(a, b)
