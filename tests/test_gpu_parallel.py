"""Partitioned assembly on the GPU: reference API invariance and slabs."""

import numpy as np
import pytest

from conftest import Golden, rel_frob

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["tri_p1_lmax3", "hex_q1_gl3"])
def test_parallel_assemble_partition_invariance(name):
    """parallel.py:128-203 contract (test_parallel.py:93-114)."""
    from paper_2101_08825_b200.parallel import parallel_assemble
    g = Golden(name)
    mesh, space, kp, cfg = g.build()
    for n_parts in (1, 2, 4):
        A, ctxs = parallel_assemble(mesh, space, kp, cfg, n_parts=n_parts)
        assert A.events == int(g["events"])
        assert sum(c.events for c in ctxs) == A.events
        assert rel_frob(A.vals, g["vals"]) <= 1e-12
        rows = np.sort(np.concatenate([c.owned_rows for c in ctxs]))
        assert np.array_equal(rows, np.arange(space.n_dofs))
        for c in ctxs:
            assert c.t_t >= c.t_a >= 0.0


@pytest.mark.parametrize("name", ["hex_q1_gl3", "tri_p1_lmax3",
                                  "quad_q2_lmax2"])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_on_one_device(name, world):
    from paper_2101_08825_b200.parallel import emulate_slabs
    g = Golden(name)
    mesh, space, kp, cfg = g.build()
    full, events = emulate_slabs(mesh, space, kp, cfg, world)
    assert events == int(g["events"])
    assert rel_frob(full.cpu().numpy(), g["vals"]) <= 1e-12


def test_assemble_distributed_single_rank(tmp_path):
    """The multi-GPU entry point on a 1-rank NCCL group equals the
    reference (scaling contract, finish path, gather)."""
    import torch
    import torch.distributed as dist
    from paper_2101_08825_b200.parallel import assemble_distributed
    g = Golden("hex_q1_gl3")
    mesh, space, kp, cfg = g.build()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg",
                            rank=0, world_size=1)
    try:
        A = assemble_distributed(mesh, space, kp, cfg)
    finally:
        dist.destroy_process_group()
    assert A.events == int(g["events"])
    assert rel_frob(A.vals, g["vals"]) <= 1e-12
