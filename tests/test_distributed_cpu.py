"""Multi-rank host logic of the z-slab path (gloo, world_size 2, CPU).

Per-rank slab partial matrices come from the CPU oracle (the checker);
the product code under test is the slab plan (row/value ranges), the
interface-plane exchange and the row-block gather of parallel.py.  The
merged result must equal the full single-process assembly bit for bit
(each shared plane is summed as own + previous, which is how the oracle's
serial scatter adds them only up to rounding order, hence the 1e-14 bound).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import Golden, rel_frob


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _golden(name):
    if name.startswith("delaunay_"):
        from test_delaunay import DGolden     # unstructured (BASELINE #2)
        return DGolden(name)
    return Golden(name)


def _worker(rank, world, port, name, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2101_08825_b200.assembly import HostPattern
        from paper_2101_08825_b200.parallel import (SlabPlan, exchange_interfaces,
                                                    gather_rows, slab_layers)
        g = _golden(name)
        mesh, space, kp, cfg = g.build()
        layers = slab_layers(mesh, world)
        A = HostPattern.for_space(mesh, space, kp, cfg)
        plans = [SlabPlan(mesh, space, A.rowptr, layers, r)
                 for r in range(world)]
        plan = plans[rank]
        inner = plan.inner_ids(mesh)
        mask = np.zeros(mesh.n_elements, np.uint8)
        mask[inner] = 1
        ev = oracle.run_general(mesh, space, kp, cfg, A, inner_mask=mask)
        a, b = plan.vals_touch
        outside = np.concatenate([A.vals[:a], A.vals[b:]])
        assert np.all(outside == 0.0), "slab wrote outside its row range"
        local = torch.from_numpy(A.vals[a:b].copy())
        exchange_interfaces(local, plan)
        full = gather_rows(local, plan, plans, A.nnz)
        evs = torch.tensor([ev], dtype=torch.int64)
        dist.all_reduce(evs)
        if rank == 0:
            out_q.put((full.numpy() * 2.0, int(evs.item()), layers))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("hex_q1_gl3", 2),
                                        ("tri_p1_lmax3", 2),
                                        ("quad_q2_lmax2", 2),
                                        ("delaunay_tri6", 2),
                                        ("delaunay_tri6", 3)])
def test_slab_exchange_and_gather_gloo(name, world, oracle_lib):
    """Delaunay slabs share dof_spill = 2 lattice planes per interface
    (their vertices sit up to two planes above the element's bin row)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    vals, events, layers = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _golden(name)
    assert events == int(g["events"])
    assert rel_frob(vals, g["vals"]) <= 1e-14
    assert layers[0][0] == 0 and layers[-1][1] > layers[0][1]


def test_slab_layers_balanced():
    from paper_2101_08825_b200 import build_mesh
    from paper_2101_08825_b200.parallel import slab_layers
    mesh = build_mesh(3, ((0, 0.5),) * 3, 1 / 32, 0.1, "hex")
    for world in (1, 2, 4, 8):
        L = slab_layers(mesh, world)
        assert L[0][0] == 0 and L[-1][1] == mesh.grid_ncells[2]
        assert all(a < b for a, b in L)
        assert all(L[i][1] == L[i + 1][0] for i in range(world - 1))
        sizes = [b - a for a, b in L]
        assert max(sizes) - min(sizes) <= 1


def test_assemble_distributed_scaling_contract():
    """assemble_distributed must not rescale: SlabAssembler.assemble_local
    runs the kernels with scale 2 (the folded _finish doubling)."""
    import inspect
    from paper_2101_08825_b200 import parallel
    src = inspect.getsource(parallel.assemble_distributed)
    assert "full * 2" not in src
    src2 = inspect.getsource(parallel.SlabAssembler.assemble_local)
    assert "scale" not in src2 or "scale=2" in src2


def _host_worker(rank, world, port, name, out_q):
    """The host-gather path of assemble_distributed: interface exchange,
    owned slices written into one node-shared array, halo windows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2101_08825_b200.assembly import HostPattern
        from paper_2101_08825_b200.parallel import (
            SharedHostArray, SlabPlan, exchange_interfaces, halo_window,
            slab_layers, window_range)
        g = _golden(name)
        mesh, space, kp, cfg = g.build()
        layers = slab_layers(mesh, world)
        A = HostPattern.for_space(mesh, space, kp, cfg)
        plans = [SlabPlan(mesh, space, A.rowptr, layers, r)
                 for r in range(world)]
        plan = plans[rank]
        mask = np.zeros(mesh.n_elements, np.uint8)
        mask[plan.inner_ids(mesh)] = 1
        oracle.run_general(mesh, space, kp, cfg, A, inner_mask=mask)
        a, b = plan.vals_touch
        local = torch.from_numpy(A.vals[a:b] * 2.0)
        exchange_interfaces(local, plan)
        shm = SharedHostArray(A.nnz)
        oa, ob = plan.vals_own
        shm.array[oa:ob] = local[oa - a:ob - a].numpy()
        win, wa = halo_window(local, plan, plans, A)
        assert (wa, wa + win.numel()) == window_range(plan, plans, A)
        dist.barrier()
        # every rank's window equals the merged matrix over that range
        full = np.array(shm.array)
        ok = bool(np.array_equal(win.numpy(), full[wa:wa + win.numel()]))
        flag = torch.tensor([int(ok)])
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            out_q.put((full, int(flag.item())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("hex_q1_gl3", 2),
                                        ("hex_q1_gl3", 3),
                                        ("tri_p1_lmax3", 2)])
def test_host_gather_and_halo_windows_gloo(name, world, oracle_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker,
                         args=(r, world, port, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    vals, ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _golden(name)
    assert ok == 1
    assert rel_frob(vals, g["vals"]) <= 1e-14
