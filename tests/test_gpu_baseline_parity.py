"""GPU vs oracle parity at the BASELINE shapes.

The golden fixtures pin the oracle to the live reference on small meshes;
these tests pin the GPU to the oracle on the headline workloads themselves,
through the reference's own partial-oracle mechanism (parallel.py:161-171:
outer = all elements, inner = a subset gives exactly the subset's pair
blocks):

  * R4 (BASELINE #4 stand-in, 474,552 hexes): one full interior cell
    layer of inner elements (6,084 hexes, ~1.8e7 pairs).  Every value of
    the two DOF planes the layer touches, and the event count, against
    the oracle;
  * R4-small ("for full parity"): the whole matrix;
  * R3-8h: a slab of four cell rows;
  * R5-tet-small (BASELINE #5 as written: jittered tets, tet11): one full
    cube layer (all six Kuhn protos).

Events must be identical (test_parallel.py:111-112 style); values within
1e-10 relative Frobenius (north star).  The oracle runs on all host cores
(oracle.run_general_tiled: tiles of one parity class in parallel, classes
in sequence, deterministic).
"""

import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _layer_parity(name, layer_offset=0, nlayers=1, first=None):
    import oracle
    import torch
    import bench
    from paper_2101_08825_b200 import _native as N
    from paper_2101_08825_b200.assembly import AssemblyContext
    mesh, space, kp, cfg = bench.build_problem(name)
    ax = mesh.dim - 1
    nl = int(mesh.grid_ncells[ax])
    z0 = nl // 2 + layer_offset
    layer = mesh.elem_cell[:, ax]
    inner = np.nonzero((layer >= z0) & (layer < z0 + nlayers))[0]
    if first is not None:
        inner = inner[:first]
    ctx = AssemblyContext(mesh, space, kp, cfg)
    A = ctx.new_matrix()
    cnt = ctx.run(A, inner_ids=inner).cpu().numpy()
    # the DOF planes the layers touch: [z0, z0 + nlayers] (degree 1)
    plane = int(np.prod(space.grid_dims[:-1]))
    a = int(A.rowptr[z0 * plane])
    b = int(A.rowptr[(z0 + nlayers + 1) * plane])
    got = A._dvals[a:b].cpu().numpy()
    outside = float(A._dvals[:a].abs().sum() + A._dvals[b:].abs().sum())
    del A
    torch.cuda.empty_cache()
    want = np.zeros(b - a)
    ev = oracle.run_general_tiled(mesh, space, kp, cfg, ctx_pattern(ctx),
                                  inner, want, base=a)
    want *= 2.0
    ptr, _ = oracle.candidates(
        mesh, kp.delta + kp.eps, np.arange(mesh.n_elements),
        np.isin(np.arange(mesh.n_elements), inner).astype(np.uint8))
    err = rel_frob(got, want)
    print(f"{name}: {len(inner)} inner elements, pairs {int(ptr[-1])}, "
          f"events {int(cnt[N.CNT_EVENTS])} / oracle {ev}, rel F {err:.2e}")
    assert int(cnt[N.CNT_PAIRS]) == int(ptr[-1])
    assert int(cnt[N.CNT_EVENTS]) == ev
    assert outside == 0.0
    assert np.linalg.norm(want) > 0
    assert err <= TOL
    return err


def ctx_pattern(ctx):
    from paper_2101_08825_b200.assembly import HostPattern, pattern_halfwidth
    K, _ = pattern_halfwidth(ctx.mesh, ctx.params, ctx.config,
                             ctx.space.degree)
    return HostPattern(ctx.space, K, allocate=False)


def test_r4_interior_layer_matches_oracle():
    """R4 headline: one full interior cell layer, exact events and every
    value of its two DOF planes."""
    _layer_parity("R4")


def test_r3_8h_slab_matches_oracle():
    _layer_parity("R3-8h", nlayers=4)


def test_r5_tet_small_layer_matches_oracle():
    """BASELINE #5 as written (jittered tets, tet11; parity vs the C
    restatement of the reference algorithm)."""
    _layer_parity("R5-tet-small")


def test_r4_small_full_matrix_matches_oracle():
    """SURVEY 8(d) "R4-small ... for full parity": the whole matrix, the
    event count and the asymmetry diagnostic."""
    import oracle
    import bench
    from paper_2101_08825_b200 import assemble
    from paper_2101_08825_b200.assembly import HostPattern
    mesh, space, kp, cfg = bench.build_problem("R4-small")
    A = assemble(mesh, space, kp, cfg)
    R = HostPattern.for_space(mesh, space, kp, cfg)
    ev = oracle.run_general_tiled(mesh, space, kp, cfg, R,
                                  np.arange(mesh.n_elements), R.vals)
    R.vals *= 2.0
    err = rel_frob(A.vals, R.vals)
    asym = oracle.asymmetry_inf(R)
    print(f"R4-small: events {A.events} / oracle {ev}, rel F {err:.2e}, "
          f"asym {A.presym_asymmetry:.6e} / {asym:.6e}")
    assert A.events == ev
    assert err <= TOL
    assert abs(A.presym_asymmetry - asym) <= 1e-9 * max(asym, 1e-300) + \
        1e-12 * float(np.abs(R.vals).max())
