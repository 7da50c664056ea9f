"""Unstructured Delaunay P1 triangle meshes (BASELINE config #2; SURVEY.md
8(f) f2).

The reference builds structured meshes only (mesh.py:153-178), but its pair
core `_general_core` (_kernels.py:391-487, `_event_tri` 146-181) is valid
for arbitrary affine triangles and takes plain arrays.  The fixtures in
tests/golden/delaunay_*.npz were produced by running that LIVE numba core
on meshes from `build_delaunay_mesh` (tests/golden/make_golden_delaunay.py),
so this element is pinned to reference arithmetic:
  * CPU: the mesh builder reproduces the fixture mesh (connectivity, bins,
    colouring); the 6-point rule is exact to degree 4; the mesh is
    conforming, oriented, region-pure, emax <= 2h, the colouring is
    vertex-disjoint; the C oracle reproduces the reference candidate lists,
    events and values bit for bit;
  * GPU (through the C-ABI): the warp-cooperative kernel k_tri_q, the
    inline row-split kernel k_tri_u (no-shortcut / eps = 0 paths) and the
    generic kernel give identical events and values within 1e-10 relative
    Frobenius norm of the reference, bit-identical run to run; partition
    invariance and the multi-GPU slab emulation; A 1 = 0 and oracle parity
    on a larger mesh; load vector and solve.
"""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, rel_frob

TOL = 1e-10
NAMES = ("delaunay_tri6", "delaunay_tri7_lmin2", "delaunay_eps0")


class DGolden:
    def __init__(self, name):
        self.z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        self.meta = json.loads(str(self.z["meta"]))

    def __getitem__(self, k):
        return self.z[k]

    def build(self):
        from paper_2101_08825_b200 import (AssemblyConfig, FESpace,
                                           KernelParams)
        from paper_2101_08825_b200.mesh import build_delaunay_mesh
        m = self.meta
        h = m["h"]
        kp = KernelParams(2, m["delta_h"] * h, m["eps_h"] * h)
        mesh = build_delaunay_mesh(m["omega"], h, kp.delta + kp.eps,
                                   jitter=m["jitter"], seed=m["seed"])
        space = FESpace(mesh, 1)
        cfg = AssemblyConfig(L_min=m["L_min"], L_max=m["L_max"],
                             outer_rule=m["rule"], inner_rule=m["rule"],
                             strategy="general")
        return mesh, space, kp, cfg


_BUILT = {}


def built(name):
    if name not in _BUILT:
        _BUILT[name] = (DGolden(name),) + DGolden(name).build()
    return _BUILT[name]


# ---------------------------------------------------------------- CPU

def test_dunavant6_exact_to_degree_4():
    from paper_2101_08825_b200.quadrature import dunavant6, rule_for_kind
    r = dunavant6()
    P, w = r.ref_points, r.weights
    assert len(r) == 6 and abs(w.sum() - 0.5) < 1e-15
    for i in range(5):
        for j in range(5 - i):
            exact = math.factorial(i) * math.factorial(j) / math.factorial(
                i + j + 2)
            got = float((w * P[:, 0] ** i * P[:, 1] ** j).sum())
            assert abs(got - exact) <= 1e-15, (i, j)
    # degree 5 is not integrated exactly (it is a degree-4 rule)
    assert abs(float((w * P[:, 0] ** 5).sum()) - 1 / 42) > 1e-6
    assert len(rule_for_kind("tri", "tri6")) == 6
    assert len(rule_for_kind("tri", "default")) == 7   # reference default
    with pytest.raises(ValueError):
        rule_for_kind("quad", "tri6")


@pytest.mark.parametrize("name", NAMES)
def test_builder_reproduces_fixture_mesh(name):
    g, mesh, space, kp, cfg = built(name)
    assert np.array_equal(mesh.nodes, g["nodes"])
    assert np.array_equal(mesh.elem_nodes, g["elem_nodes"])
    assert np.array_equal(mesh.elem_cell, g["elem_cell"])
    assert np.array_equal(mesh.elem_color, g["elem_color"])
    assert np.array_equal(mesh.elem_region, g["elem_region"])
    assert np.array_equal(space.free, g["free"])


@pytest.mark.parametrize("jitter,seed", [(0.0, 0), (0.3, 0), (0.35, 5)])
def test_delaunay_mesh_properties(jitter, seed):
    from paper_2101_08825_b200.mesh import build_delaunay_mesh
    h = 1 / 32
    mesh = build_delaunay_mesh(((0.0, 0.25), (0.0, 0.375)), h, 0.1,
                               jitter=jitter, seed=seed)
    c = mesh.elem_coords
    det = ((c[:, 1, 0] - c[:, 0, 0]) * (c[:, 2, 1] - c[:, 0, 1])
           - (c[:, 1, 1] - c[:, 0, 1]) * (c[:, 2, 0] - c[:, 0, 0]))
    assert (det > 0).all()
    # the triangles tile the whole box [origin, origin + nc h]
    lo = np.asarray(mesh.grid_origin)
    hi = lo + np.asarray(mesh.grid_ncells) * h
    assert abs(0.5 * det.sum() - np.prod(hi - lo)) < 1e-12
    # and so does Omega (region purity)
    om = mesh.elem_region == 0
    assert abs(0.5 * det[om].sum() - 0.25 * 0.375) < 1e-12
    # conforming: every interior edge is shared by exactly two triangles
    e = np.sort(np.concatenate([mesh.elem_nodes[:, [0, 1]],
                                mesh.elem_nodes[:, [1, 2]],
                                mesh.elem_nodes[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e[:, 0] * len(mesh.nodes) + e[:, 1],
                       return_counts=True)
    assert set(np.unique(cnt)) <= {1, 2}
    assert mesh.emax <= 2.0 * h
    assert np.allclose(mesh.elem_lo, c.min(axis=1))
    # bins: lower corner inside the element's cell, bin-lex order
    cell = mesh.elem_cell
    rel = (mesh.elem_lo - lo) / h
    assert ((rel >= cell - 1e-12) & (rel < cell + 1 + 1e-12)).all()
    flat = cell[:, 1].astype(np.int64) * mesh.grid_ncells[0] + cell[:, 0]
    assert (np.diff(flat) >= 0).all()
    # the colouring is vertex-disjoint
    for k in range(mesh.n_colors):
        v = mesh.elem_nodes[mesh.elem_color == k].ravel()
        assert len(np.unique(v)) == len(v)
    # vertices keep their lattice node: |x - node| <= jitter h
    nv = np.asarray(mesh.grid_ncells) + 1
    ids = np.arange(len(mesh.nodes))
    g = np.stack([ids % nv[0], ids // nv[0]], axis=1)
    assert np.abs(mesh.nodes - (lo + g * h)).max() <= jitter * h + 1e-15


def test_delaunay_space_and_pattern():
    from paper_2101_08825_b200 import AssemblyConfig, FESpace, KernelParams
    from paper_2101_08825_b200.assembly import HostPattern, resolve_strategy
    g, mesh, space, kp, cfg = built("delaunay_tri6")
    assert space.n_dofs == len(mesh.nodes)
    assert np.array_equal(space.element_dofs, mesh.elem_nodes)
    # constrained = not strictly inside Omega (exact lattice test)
    x = space.dof_coords
    inside = np.all((x > 0.0) & (x < 0.25), axis=1)
    assert np.array_equal(np.nonzero(inside)[0], space.free)
    A = HostPattern.for_space(mesh, space, kp, cfg)
    assert np.array_equal(A.rowptr, g["rowptr"]) and A.K == int(g["K"])
    assert resolve_strategy(mesh, AssemblyConfig()) == "general"
    with pytest.raises(ValueError):
        resolve_strategy(mesh, AssemblyConfig(strategy="blocked"))
    with pytest.raises(ValueError):
        FESpace(mesh, 2)
    with pytest.raises(ValueError):
        KernelParams(2, 0.1, 0.1)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_core(name, oracle_lib):
    g, mesh, space, kp, cfg = built(name)
    n = mesh.n_elements
    ptr, ids = oracle_lib.candidates(mesh, kp.delta + kp.eps,
                                     np.arange(n, dtype=np.int64),
                                     np.ones(n, np.uint8))
    assert np.array_equal(ptr, g["cand_ptr"])
    assert np.array_equal(ids, g["cand_ids"])
    R = oracle_lib.assemble_general(mesh, space, kp, cfg)
    assert R.events == int(g["events"])
    assert np.array_equal(R.vals, g["vals"])
    assert R.presym_asymmetry == float(g["asym"])
    # A 1 = 0 (test_assembly.py:49-55)
    rs = np.add.reduceat(R.vals, R.rowptr[:-1])
    assert np.abs(rs).max() <= 1e-12 * np.abs(R.vals).max()


def test_candidates_cover_brute_force(oracle_lib):
    """The binned stencil finds every element pair with box gap < reach."""
    g, mesh, space, kp, cfg = built("delaunay_tri6")
    reach = kp.delta + kp.eps
    lo, hi = mesh.elem_lo, mesh.elem_hi
    gap = np.maximum(lo[:, None, :] - hi[None, :, :],
                     lo[None, :, :] - hi[:, None, :]).max(axis=2)
    want = np.maximum(gap, 0.0) < reach
    ptr, ids = g["cand_ptr"], g["cand_ids"]
    got = np.zeros_like(want)
    for l in range(mesh.n_elements):
        got[l, ids[ptr[l]:ptr[l + 1]]] = True
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, 1, 2])
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference(name, flags):
    """flags 0: row-split k_tri_u; 1: generic kernel; 2: no shortcuts."""
    from paper_2101_08825_b200 import assemble
    g, mesh, space, kp, cfg = built(name)
    A = assemble(mesh, space, kp, cfg, flags=flags)
    assert np.array_equal(A.rowptr, g["rowptr"]) and A.K == int(g["K"])
    assert A.events == int(g["events"])
    err = rel_frob(A.vals, g["vals"])
    print(f"{name} flags={flags}: events={A.events} relF={err:.3e}")
    assert err <= TOL
    assert abs(A.presym_asymmetry - float(g["asym"])) <= 1e-9 * np.abs(
        g["vals"]).max()


@pytest.mark.gpu
def test_gpu_neighbor_lists_and_determinism():
    from paper_2101_08825_b200 import assemble, neighbor_sets
    g, mesh, space, kp, cfg = built("delaunay_tri6")
    ns = neighbor_sets(mesh, kp)
    assert np.array_equal(ns.ptr, g["cand_ptr"])
    assert np.array_equal(ns.ids, g["cand_ids"])
    a = assemble(mesh, space, kp, cfg).vals
    b = assemble(mesh, space, kp, cfg).vals
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_gpu_partitions_and_slabs():
    from paper_2101_08825_b200.parallel import emulate_slabs, parallel_assemble
    g, mesh, space, kp, cfg = built("delaunay_tri6")
    for n_parts in (2, 3):
        A, _ = parallel_assemble(mesh, space, kp, cfg, n_parts=n_parts)
        assert A.events == int(g["events"])
        assert rel_frob(A.vals, g["vals"]) <= 1e-12
    for world in (2, 3):
        full, events = emulate_slabs(mesh, space, kp, cfg, world)
        assert events == int(g["events"])
        assert rel_frob(full.cpu().numpy(), g["vals"]) <= 1e-12


def _r2_small():
    """BASELINE #2 parameters on Omega = [0, 0.25]^2 (h = 1/400,
    delta = 0.05, eps = h/2, 6-point rule, L_max = 3)."""
    from paper_2101_08825_b200 import AssemblyConfig, FESpace, KernelParams
    from paper_2101_08825_b200.mesh import build_delaunay_mesh
    h = 1 / 400
    kp = KernelParams(2, 0.05, h / 2)
    mesh = build_delaunay_mesh(((0.0, 0.25), (0.0, 0.25)), h,
                               kp.delta + kp.eps, jitter=0.3, seed=0)
    cfg = AssemblyConfig(L_max=3, outer_rule="tri6", inner_rule="tri6",
                         strategy="general")
    return mesh, FESpace(mesh, 1), kp, cfg


@pytest.mark.gpu
def test_gpu_r2_small_vs_oracle_sample(oracle_lib):
    """R2-small (122k triangles) on the GPU; oracle rows for a seeded
    sample of inner elements (the reference's slab mechanism,
    parallel.py:161-171: outer = all, inner = sample) must match the GPU
    values on the rows only those elements touch, and A 1 = 0."""
    from paper_2101_08825_b200 import assemble
    from paper_2101_08825_b200.assembly import HostPattern
    mesh, space, kp, cfg = _r2_small()
    A = assemble(mesh, space, kp, cfg)
    rs = np.add.reduceat(A.vals, A.rowptr[:-1])
    assert np.abs(rs).max() <= 1e-11 * np.abs(A.vals).max()
    assert A.presym_asymmetry <= 1e-2 * np.abs(A.vals).max()
    rng = np.random.default_rng(0)
    # a vertex patch: every element around 6 seeded vertices
    verts = rng.choice(np.nonzero(space.constrained_mask == 0)[0], 6,
                       replace=False)
    inner = np.nonzero(np.isin(mesh.elem_nodes, verts).any(axis=1))[0]
    mask = np.zeros(mesh.n_elements, np.uint8)
    mask[inner] = 1
    R = HostPattern.for_space(mesh, space, kp, cfg)
    oracle_lib.run_general(mesh, space, kp, cfg, R, inner_mask=mask)
    R.vals *= 2.0
    for r in verts:        # rows whose elements are all in the sample
        a, b = A.rowptr[r], A.rowptr[r + 1]
        err = rel_frob(A.vals[a:b], R.vals[a:b])
        assert err <= TOL, (r, err)


@pytest.mark.gpu
def test_gpu_rhs_and_solve():
    """Manufactured u = x^2 + y^2, f = -4 (exact for the nonlocal operator,
    harness.py:92-95): load vector vs a host restatement, GPU solve vs a
    CPU solve of the reference-core matrix, and a small L2 error."""
    import scipy.sparse.linalg as spla
    from paper_2101_08825_b200 import assemble, assemble_rhs, solve
    from paper_2101_08825_b200.fe_space import l2_error
    from paper_2101_08825_b200.quadrature import dunavant7
    g, mesh, space, kp, cfg = built("delaunay_tri6")
    A = assemble(mesh, space, kp, cfg)
    f = lambda x: -4.0 + 0.0 * x[..., 0]
    u_ex = lambda x: (x ** 2).sum(axis=-1)
    rhs = assemble_rhs(mesh, space, kp, f, u_ex, A)
    r = dunavant7()
    load = np.zeros(space.n_dofs)
    for e in mesh.omega_element_ids():
        v = mesh.elem_coords[e]
        E = np.column_stack([v[1] - v[0], v[2] - v[0]])
        det = abs(np.linalg.det(E))
        pts = v[0] + r.ref_points @ E.T
        lam = np.column_stack([1 - r.ref_points.sum(axis=1), r.ref_points])
        load[space.element_dofs[e]] += det * (r.weights * f(pts)) @ lam
    gt = np.zeros(space.n_dofs)
    gt[space.constrained] = u_ex(space.dof_coords[space.constrained])
    S = A.to_scipy()
    S.data = g["vals"].copy()
    want = (load - S @ gt)[space.free]
    assert np.abs(rhs - want).max() <= 1e-9 * np.abs(want).max()
    u, rep = solve(A, rhs, space.free, space.constrained,
                   u_ex(space.dof_coords[space.constrained]))
    assert rep.converged
    Aff = S[space.free][:, space.free]
    ref = spla.spsolve(Aff.tocsc(), want)
    assert np.abs(u[space.free] - ref).max() <= 1e-8 * max(
        1.0, np.abs(ref).max())
    assert l2_error(space, u, u_ex) <= 5e-3


@pytest.mark.gpu
@pytest.mark.parametrize("lmin,lmax", [(1, 1), (1, 2), (2, 2), (3, 3)])
def test_gpu_recursion_windows_vs_oracle(lmin, lmax, oracle_lib):
    """Other [L_min, L_max] windows on the fixture mesh (the k_tri_q walk
    has separate code for L_max 1/2/3 and forced splits), against the
    oracle, which reproduces the reference core bit for bit on the
    fixtures (test_oracle_matches_reference_core)."""
    from paper_2101_08825_b200 import AssemblyConfig, assemble
    g, mesh, space, kp, _ = built("delaunay_tri6")
    cfg = AssemblyConfig(L_min=lmin, L_max=lmax, outer_rule="tri6",
                         inner_rule="tri6", strategy="general")
    A = assemble(mesh, space, kp, cfg)
    R = oracle_lib.assemble_general(mesh, space, kp, cfg)
    assert A.events == R.events
    assert rel_frob(A.vals, R.vals) <= TOL


def test_strang3_exact_to_degree_2():
    from paper_2101_08825_b200.quadrature import rule_for_kind, strang3
    r = strang3()
    P, w = r.ref_points, r.weights
    for i in range(3):
        for j in range(3 - i):
            exact = math.factorial(i) * math.factorial(j) / math.factorial(
                i + j + 2)
            assert abs(float((w * P[:, 0] ** i * P[:, 1] ** j).sum())
                       - exact) <= 1e-15
    assert len(rule_for_kind("tri", "tri3")) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("flags", [0, 4])
def test_gpu_tri3_rule_vs_oracle(flags, oracle_lib):
    """The 3-point rule of BASELINE config #1 as written ("tri3"), on the
    structured R1-type mesh (row-split kernel; flags 4 -> the generic
    kernel, k_2d is Dunavant-7 only) and on a Delaunay mesh."""
    from paper_2101_08825_b200 import (AssemblyConfig, FESpace, KernelParams,
                                       assemble, build_mesh)
    h = 1 / 32
    kp = KernelParams(2, 0.1, h / 2)
    cfg = AssemblyConfig(L_max=3, outer_rule="tri3", inner_rule="tri3",
                         strategy="general")
    mesh = build_mesh(2, ((0.0, 0.5), (0.0, 0.5)), h, kp.delta + kp.eps,
                      "tri")
    space = FESpace(mesh, 1)
    A = assemble(mesh, space, kp, cfg, flags=flags)
    R = oracle_lib.assemble_general(mesh, space, kp, cfg)
    assert A.events == R.events and rel_frob(A.vals, R.vals) <= TOL
    g, dmesh, dspace, dkp, _ = built("delaunay_tri6")
    A = assemble(dmesh, dspace, dkp, cfg, flags=flags)
    R = oracle_lib.assemble_general(dmesh, dspace, dkp, cfg)
    assert A.events == R.events and rel_frob(A.vals, R.vals) <= TOL
