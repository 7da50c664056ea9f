"""Partitioned assembly: the reference API on one device, z-slabs over ranks.

Two layers:

1. `parallel_assemble` / `ghost_regions` / `PartitionContext` restate the
   reference's partitioned assembly (parallel.py:38-203): RCB partitions
   (mesh.partition_geometric), ghost outer regions Gamma_JI, row ownership
   by the lowest-id element, a private value buffer per partition and a
   fixed-order merge.  Each partition runs the device kernel with
   outer = owned + ghosts and inner = owned, exactly the reference's
   `_run_general(outer_ids, inner_mask)` call.

2. `SlabAssembler` is the multi-GPU path: one process per GPU
   (torch.distributed), inner elements split into z-slabs of whole cell
   layers balanced by pair count.  All of a pair's entries land in rows of
   its inner element (_kernels.py:483-486), so rank r writes only the DOF
   planes of its layers; those rows are a contiguous range of the
   implicit pattern (DOF ids are z-major), so each rank allocates only its
   row block.  The shared DOF plane(s) between consecutive slabs (one on
   structured meshes, `dof_spill` on Delaunay meshes) are
   summed with one send/recv per interface (rank r -> r+1, added in rank
   order), after which every rank owns a disjoint row block; `gather`
   collects the blocks on rank 0 (NCCL has no gatherv, so grouped
   send/recv).  No collective touches the pair computation itself.

The communication code is device-agnostic (NCCL tensors on GPUs, gloo on
CPU for the world_size-2 tests).
"""

import time

import numpy as np

from . import _native as N
from .assembly import (AssemblyConfig, AssemblyContext, SparseMatrix,
                       pattern_halfwidth)
from .mesh import partition_geometric

__all__ = ["PartitionContext", "ghost_regions", "parallel_assemble",
           "slab_layers", "SlabAssembler"]


# ---------------------------------------------------------------------------
# reference API (parallel.py:38-203)

class PartitionContext:
    """owned elements, owned rows, ghosts {J: ids}, timers and events."""

    def __init__(self, part, owned, owned_rows, ghosts):
        self.part = part
        self.owned = owned
        self.owned_rows = owned_rows
        self.ghosts = ghosts
        self.t_a = 0.0
        self.t_t = 0.0
        self.events = 0

    @property
    def n_outer(self):
        return self.owned.size + sum(g.size for g in self.ghosts.values())

    def __repr__(self):
        return (f"PartitionContext(part={self.part}, owned={self.owned.size},"
                f" ghost={sum(g.size for g in self.ghosts.values())})")


def ghost_regions(mesh, partition_map, params):
    """{(J, I): Gamma_JI}: J-owned elements within box distance delta+eps
    of part I's bounding box; (I, I) is I's constraint-layer part."""
    reach = params.delta + params.eps
    owner = partition_map.owner
    out = {}
    for ip in range(partition_map.n_parts):
        box = partition_map.part_bbox[ip]
        gap = np.maximum(np.maximum(mesh.elem_lo - box.hi,
                                    box.lo - mesh.elem_hi), 0.0).max(axis=1)
        near = gap < reach
        for jp in range(partition_map.n_parts):
            if jp == ip:
                out[(ip, ip)] = np.nonzero((owner == ip)
                                           & (mesh.elem_region == 1))[0]
            else:
                out[(jp, ip)] = np.nonzero(near & (owner == jp))[0]
    return out


def _row_owner(mesh, space, partition_map):
    """Row r belongs to the part owning the lowest-id element holding r."""
    n = mesh.n_elements
    first = np.full(space.n_dofs, n, dtype=np.int64)
    ed = space.element_dofs
    for j in range(ed.shape[1]):
        col = ed[:, j]
        ok = col >= 0
        np.minimum.at(first, col[ok], np.arange(n)[ok])
    if first.max() >= n:
        raise AssertionError("dangling DOF without an element")
    return partition_map.owner[first]


def parallel_assemble(mesh, space, kernel, config=None, n_parts=1,
                      partition_map=None, device=None):
    """Assemble A = 2(A21 + A22) over n_parts partitions (parallel.py:128).

    Returns (A, contexts).  Partitions run one after another on the device
    (each is a full-width GPU launch); the merge sums the private buffers
    per row owner in partition order.
    """
    import torch
    config = config or AssemblyConfig()
    if config.method != "mollified_adaptive":
        raise ValueError("parallel assembly supports the adaptive method only")
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    if partition_map is None:
        partition_map = partition_geometric(mesh, n_parts)
    regions = ghost_regions(mesh, partition_map, kernel)
    ctx = AssemblyContext(mesh, space, kernel, config, device)
    row_owner = _row_owner(mesh, space, partition_map)
    contexts = []
    for ip in range(n_parts):
        owned = partition_map.owned(ip)
        ghosts = {jp: regions[(jp, ip)] for jp in range(n_parts) if jp != ip}
        contexts.append(PartitionContext(ip, owned,
                                         np.nonzero(row_owner == ip)[0],
                                         ghosts))
    t_start = time.perf_counter()
    buffers = []
    for c in contexts:
        t0 = time.perf_counter()
        outer = c.owned
        if c.ghosts:
            outer = np.sort(np.concatenate(
                [outer] + [g for g in c.ghosts.values() if g.size]))
        om = np.zeros(mesh.n_elements, np.uint8)
        om[outer] = 1
        B = ctx.new_matrix()
        cnt = ctx.run(B, outer_mask=om, inner_ids=c.owned, scale=1.0)
        torch.cuda.synchronize()
        c.events = int(cnt[0].item())
        c.t_a = time.perf_counter() - t0
        buffers.append(B._dvals)
    # ownership audit: a buffer only holds rows of its own elements' DOFs
    A = ctx.new_matrix()
    rowptr = A.rowptr
    entry_owner = torch.from_numpy(
        np.repeat(row_owner, np.diff(rowptr))).to(A._dvals.device)
    for c in contexts:
        own = np.unique(space.element_dofs[c.owned])
        rows_mask = np.zeros(space.n_dofs, bool)
        rows_mask[own[own >= 0]] = True
        touched = torch.nonzero(buffers[c.part] != 0).flatten().cpu().numpy()
        if touched.size:
            rows = np.searchsorted(rowptr, touched, side="right") - 1
            if not rows_mask[rows].all():
                raise AssertionError("partition wrote a row outside its "
                                     "elements")
    # merge: one pass per row owner, buffers summed in partition order
    for c in contexts:
        sel = entry_owner == c.part
        acc = buffers[0][sel].clone()
        for jp in range(1, n_parts):
            acc += buffers[jp][sel]
        A._dvals[sel] = acc
        c.t_t = time.perf_counter() - t_start
    A._dvals *= 2.0
    counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64,
                           device=A._dvals.device)
    counters[0] = sum(c.events for c in contexts)
    ctx.finish(A, counters)
    from .assembly import _d2h
    A._vals = _d2h(A._dvals)
    return A, contexts


# ---------------------------------------------------------------------------
# z-slab multi-GPU path

def slab_layers(mesh, world, weights=None):
    """Cut the top-axis cell layers into `world` contiguous slabs.

    weights: per-element work (e.g. pair counts); slabs are balanced by
    their sum.  Returns a list of (layer_lo, layer_hi) half-open ranges.
    """
    axis = mesh.dim - 1
    layer = mesh.elem_cell[:, axis].astype(np.int64)
    nl = int(mesh.grid_ncells[axis])
    if world > nl:
        raise ValueError("more ranks than cell layers")
    w = np.bincount(layer, weights=weights, minlength=nl).astype(float)
    cum = np.cumsum(w)
    total = cum[-1] if cum[-1] > 0 else 1.0
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, total * r / world, side="left")) + 1
        c = max(c, cuts[-1] + 1)
        c = min(c, nl - (world - r))
        cuts.append(c)
    cuts.append(nl)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def slab_layers_fracs(mesh, fracs, weights=None):
    """Contiguous top-axis layer ranges whose cumulative work reaches the
    given fractions (ascending, last = 1.0), at least one layer each."""
    axis = mesh.dim - 1
    layer = mesh.elem_cell[:, axis].astype(np.int64)
    nl = int(mesh.grid_ncells[axis])
    w = np.bincount(layer, weights=weights, minlength=nl).astype(float)
    cum = np.cumsum(w)
    total = cum[-1] if cum[-1] > 0 else 1.0
    cuts = [0]
    k = len(fracs)
    for r, f in enumerate(fracs[:-1], start=1):
        c = int(np.searchsorted(cum, total * f, side="left")) + 1
        c = max(c, cuts[-1] + 1)
        c = min(c, nl - (k - r))
        cuts.append(c)
    cuts.append(nl)
    return [(cuts[r], cuts[r + 1]) for r in range(k)]


class SlabPlan:
    """Rows / value ranges of one rank's slab on the implicit pattern."""

    def __init__(self, mesh, space, rowptr, layers, rank):
        self.world = len(layers)
        self.rank = rank
        d = space.degree
        dims = space.grid_dims
        plane = int(np.prod(dims[:-1]))       # DOFs per top-axis plane
        nplanes = int(dims[-1])
        lo, hi = layers[rank]
        self.layers = (lo, hi)
        # an element of cell layer c touches DOF planes [d*c, d*c + spill]:
        # spill = d on structured meshes; on Delaunay meshes vertices may
        # sit up to mesh.dof_spill lattice planes above the element's bin
        spill = int(getattr(mesh, "dof_spill", d))
        self.spill = spill
        # DOF planes touched by this slab's elements: [d*lo, d*(hi-1)+spill]
        self.touch_planes = (d * lo, min(d * (hi - 1) + spill, nplanes - 1))
        # owned planes: [d*lo, d*hi) ; the last rank also owns the top
        own_hi = d * hi if rank < self.world - 1 else nplanes
        self.own_planes = (d * lo, own_hi)
        self.plane = plane
        self.rows_touch = (self.touch_planes[0] * plane,
                           (self.touch_planes[1] + 1) * plane)
        self.rows_own = (self.own_planes[0] * plane, self.own_planes[1] * plane)
        self.vals_touch = (int(rowptr[self.rows_touch[0]]),
                           int(rowptr[self.rows_touch[1]]))
        self.vals_own = (int(rowptr[self.rows_own[0]]),
                         int(rowptr[self.rows_own[1]]))
        # the planes shared with the next rank: its first spill - d + 1
        # owned planes (one plane on structured meshes)
        nshare = spill - d + 1
        if rank < self.world - 1:
            nxt_hi = layers[rank + 1][1]
            if d * hi + nshare > (d * nxt_hi if rank + 1 < self.world - 1
                                  else nplanes):
                raise ValueError("slab too thin for the element spill")
            p = d * hi
            self.send_range = (int(rowptr[p * plane]),
                               int(rowptr[(p + nshare) * plane]))
        else:
            self.send_range = None
        if rank > 0:
            p = d * lo
            self.recv_range = (int(rowptr[p * plane]),
                               int(rowptr[(p + nshare) * plane]))
        else:
            self.recv_range = None

    def inner_ids(self, mesh):
        layer = mesh.elem_cell[:, mesh.dim - 1]
        lo, hi = self.layers
        return np.nonzero((layer >= lo) & (layer < hi))[0]


def exchange_interfaces(local, plan, group=None):
    """Add the previous rank's contribution to our first owned plane.

    `local` holds this rank's touched value range (plan.vals_touch).  Rank
    r sends its top shared plane to r+1; r+1 adds it.  Ring-free and
    deterministic: every plane gets exactly (own + previous) in that order.
    """
    import torch.distributed as dist
    base = plan.vals_touch[0]
    ops = []
    recv = None
    if plan.send_range is not None:
        a, b = plan.send_range
        ops.append(dist.P2POp(dist.isend, local[a - base:b - base].contiguous(),
                              plan.rank + 1, group))
    if plan.recv_range is not None:
        a, b = plan.recv_range
        recv = local.new_empty(b - a)
        ops.append(dist.P2POp(dist.irecv, recv, plan.rank - 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    if recv is not None:
        a, b = plan.recv_range
        local[a - base:b - base] += recv
    return local


def gather_rows(local, plan, plans, nnz, group=None, dst=0):
    """Owned row blocks of every rank -> full value array on rank `dst`.

    NCCL has no gatherv, so this is one send per rank and the matching
    receives on `dst`, each straight into its slice of the full array."""
    import torch.distributed as dist
    base = plan.vals_touch[0]
    a, b = plan.vals_own
    mine = local[a - base:b - base]
    if plan.rank != dst:
        dist.send(mine.contiguous(), dst, group)
        return None
    full = local.new_empty(nnz)
    full[a:b] = mine
    for p in plans:
        if p.rank == dst:
            continue
        pa, pb = p.vals_own
        dist.recv(full[pa:pb], p.rank, group)
    return full


class SlabAssembler:
    """One rank's share of a multi-GPU assembly (see module docstring)."""

    def __init__(self, mesh, space, kernel, config, rank, world, device=None,
                 weights=None, layers=None):
        import torch
        from .device import ColorPlan
        self.rank, self.world = rank, world
        self.ctx = AssemblyContext(mesh, space, kernel, config, device)
        self.layers = layers or slab_layers(mesh, world, weights)
        K, oe = pattern_halfwidth(mesh, kernel, config, space.degree)
        self.A = SparseMatrix(space, K, allocate=False)
        self.A._offset_reach = oe
        self.plans = [SlabPlan(mesh, space, self.A.rowptr, self.layers, r)
                      for r in range(world)]
        self.plan = self.plans[rank]
        from .device import to_device
        self.A._drowptr = to_device(self.A.rowptr, self.ctx.device)
        a, b = self.plan.vals_touch
        self.local = torch.zeros(b - a, dtype=torch.float64,
                                 device=self.ctx.device)
        self.inner = self.plan.inner_ids(mesh)
        # heaviest elements first inside each colour (as the single-GPU
        # default plan) when the caller has the pair-count weights
        self.color_plan = ColorPlan(mesh, self.inner, self.ctx.device,
                                    work=weights)
        self.counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64,
                                    device=self.ctx.device)

    def assemble_local(self):
        """Pairs of this slab's inner elements into the local row block."""
        from .assembly import WindowedValues
        self.local.zero_()
        self.counters.zero_()
        win = WindowedValues(self.local, self.plan.vals_touch[0])
        self.ctx.run(self.A, plan=self.color_plan, counters=self.counters,
                     vals_window=win)
        return self.counters

    def exchange(self, group=None):
        return exchange_interfaces(self.local, self.plan, group)

    def gather(self, group=None, dst=0):
        return gather_rows(self.local, self.plan, self.plans, self.A.nnz,
                           group, dst)


def emulate_slabs(mesh, space, kernel, config, world, device=None):
    """Run every rank's slab on ONE device, one after another, and merge
    with the same interface/gather arithmetic (tests and single-GPU runs
    of the multi-GPU decomposition; ranks never wait on each other)."""
    import torch
    ranks = [SlabAssembler(mesh, space, kernel, config, r, world, device)
             for r in range(world)]
    events = 0
    for s in ranks:
        events += int(s.assemble_local()[0].item())
    # interface planes: rank r's shared top plane is added into rank r+1
    for r in range(world - 1):
        src, dst = ranks[r], ranks[r + 1]
        a, b = src.plan.send_range
        ra, rb = dst.plan.recv_range
        assert (a, b) == (ra, rb)
        dst.local[ra - dst.plan.vals_touch[0]:rb - dst.plan.vals_touch[0]] += \
            src.local[a - src.plan.vals_touch[0]:b - src.plan.vals_touch[0]]
    full = torch.empty(ranks[0].A.nnz, dtype=torch.float64,
                       device=ranks[0].local.device)
    for s in ranks:
        a, b = s.plan.vals_own
        base = s.plan.vals_touch[0]
        full[a:b] = s.local[a - base:b - base]
    return full, events


def pair_counts(mesh, params, dmesh):
    """Candidate-pair count per element (the count pass of the GPU
    neighbour search, mf_count_candidates) -- the slab balancing weight."""
    import ctypes

    import torch

    from . import _native as N
    from .assembly import stencil_pad, stencil_radius
    n = mesh.n_elements
    dev = dmesh.device
    outer = torch.arange(n, dtype=torch.int64, device=dev)
    mask = torch.ones(n, dtype=torch.uint8, device=dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    reach = params.delta + params.eps
    N.check(N.lib().mf_count_candidates(
        ctypes.byref(dmesh.struct), N.ptr(outer), n, N.ptr(mask),
        stencil_radius(reach + stencil_pad(mesh), mesh.h), float(reach),
        N.ptr(counts),
        N.stream_ptr()), "mf_count_candidates")
    return counts.cpu().numpy()


def assemble_distributed(mesh, space, kernel, config=None, group=None,
                         dst=0, weights=None):
    """Multi-GPU `assemble`: every rank of the process group calls it with
    the same host inputs; rank `dst` returns the full SparseMatrix (host
    values, events, presym_asymmetry), the others return None."""
    import torch
    import torch.distributed as dist

    from .assembly import _d2h
    config = config or AssemblyConfig()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    s = SlabAssembler(mesh, space, kernel, config, rank, world, dev,
                      weights=weights)
    cnt = s.assemble_local().clone()
    s.exchange(group)
    full = s.gather(group, dst)
    dist.all_reduce(cnt, group=group)
    if rank != dst:
        return None
    A = s.A
    A._dvals = full          # the slab kernels already fold _finish's x2
    s.ctx.finish(A, cnt)
    A._vals = _d2h(A._dvals)
    return A
