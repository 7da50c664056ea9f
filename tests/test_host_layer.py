"""Host layer (mesh, FE space, rules, kernel constants) vs the reference.

The golden fixtures hold the reference's own mesh/FE arrays
(tests/golden/make_golden.py); equality here is bit-for-bit.  Constant
anchors are the reference's frozen values (test_kernel.py:18-70).
"""

import math

import numpy as np
import pytest

from conftest import Golden, golden_names
from paper_2101_08825_b200 import (KernelParams, build_mesh, dunavant7,
                                   gauss_legendre_1d, gauss_lobatto_1d,
                                   partition_geometric, rule_for_kind,
                                   scaling_c_delta, scaling_c_delta_eps, xi)
from paper_2101_08825_b200.assembly import (AssemblyConfig, HostPattern,
                                            aprx_max_dist, aprx_min_dist)
from paper_2101_08825_b200.mesh import BoundingBox


@pytest.mark.parametrize("name", golden_names())
def test_mesh_and_space_match_reference(name):
    g = Golden(name)
    mesh, space, kp, cfg = g.build()
    for k in ("elem_kind", "elem_proto", "elem_region", "elem_cell",
              "elem_coords", "elem_lo", "elem_hi"):
        a, b = getattr(mesh, k), g[k]
        assert a.dtype == b.dtype and np.array_equal(a, b), k
    assert np.array_equal(space.element_dofs, g["dofs"])
    assert np.array_equal(space.element_nloc, g["nloc"])
    assert np.array_equal(space.free, g["free"])
    assert kp.c_delta_eps == float(g["c_delta_eps"])
    A = HostPattern.for_space(mesh, space, kp, cfg)
    assert A.K == int(g["K"])
    assert np.array_equal(A.rowptr, g["rowptr"])


def test_kernel_anchor_values():
    assert abs(xi(np.array([0.5]))[0] - 0.9510726928710938) <= 1e-15
    assert xi(1.0) == 1.0 and xi(-1.0) == 0.0 and xi(0.0) == 0.5
    assert abs(scaling_c_delta(2, 0.2) - 795.7747154594768) <= 1e-9
    assert abs(scaling_c_delta(3, 0.2) - 3730.193978716296) <= 1e-8
    assert abs(scaling_c_delta_eps(2, 0.2, 0.1)
               - scaling_c_delta(2, 0.2) / 1.1376748251748252) <= 1e-9
    assert abs(scaling_c_delta_eps(3, 0.2, 0.1)
               - scaling_c_delta(3, 0.2) / 1.2338286713286713) <= 1e-8
    # BASELINE config #4: gamma = 15/(2 pi delta^5) is kappa = 2
    kp = KernelParams(3, 0.1, 1 / 128, kappa=2.0)
    assert kp.c_delta == pytest.approx(15 / (2 * math.pi * 0.1 ** 5),
                                       rel=1e-14)


def test_kernel_params_validation():
    for args in ((1, 0.2), (2, -0.1), (2, 0.2, 0.2), (2, 0.2, 0.0, 0.0)):
        with pytest.raises(ValueError):
            KernelParams(*args)


def test_rules():
    assert abs(dunavant7().weights.sum() - 0.5) <= 1e-15
    for n in range(1, 11):
        assert abs(gauss_legendre_1d(n).weights.sum() - 2.0) <= 1e-14
    for n in range(2, 7):
        r = gauss_lobatto_1d(n)
        assert r.ref_points[0, 0] == -1.0 and r.ref_points[-1, 0] == 1.0
    assert len(rule_for_kind("hex", "gauss2")) == 8
    assert len(rule_for_kind("tri", "gauss9")) == 7
    with pytest.raises(ValueError):
        rule_for_kind("quad", "gauss11")


def test_distance_worked_examples():
    a = BoundingBox((0.0, 0.0), (1.0, 1.0))
    b = BoundingBox((2.0, 0.0), (3.0, 1.0))
    c = BoundingBox((2.0, 5.0), (3.0, 6.0))
    assert aprx_min_dist(a, b) == 1.0
    assert abs(aprx_max_dist(a, b) - np.sqrt(10.0)) <= 1e-14
    assert aprx_min_dist(a, a) == 0.0
    assert aprx_min_dist(a, c) == 4.0
    assert abs(aprx_max_dist(a, c) - np.sqrt(45.0)) <= 1e-14


def test_mesh_validation_and_counts():
    om = ((-0.6, 0.6), (-0.4, 0.4))
    assert build_mesh(2, om, 0.1, 0.2125, "quad").n_elements == 18 * 14
    assert build_mesh(2, om, 0.1, 0.2125, "mixed").n_elements == 126 + 252
    assert build_mesh(2, om, 0.1, 0.2, "quad").gamma_layers == 2
    for bad in ((2, om, 0.07, 0.2), (2, om, -0.1, 0.2)):
        with pytest.raises(ValueError):
            build_mesh(*bad)
    with pytest.raises(ValueError):
        build_mesh(2, om, 0.1, 0.2, "hex")
    with pytest.raises(ValueError):
        AssemblyConfig(L_min=3, L_max=2)
    with pytest.raises(ValueError):
        AssemblyConfig(L_max=25)


@pytest.mark.parametrize("name", ["tri_p1_lmax3", "hex_q1_gl3"])
def test_partition_matches_reference(name):
    g = Golden(name)
    if "part_owner" not in g:
        pytest.skip("no partition data")
    mesh, *_ = g.build()
    assert np.array_equal(partition_geometric(mesh, 2).owner, g["part_owner"])


def test_r4_mesh_builds_fast():
    import time
    t = time.perf_counter()
    mesh = build_mesh(3, ((0.0, 1.0),) * 3, 1 / 64, 0.1 + 1 / 128, "hex")
    assert mesh.n_elements == 78 ** 3
    assert time.perf_counter() - t < 20.0
