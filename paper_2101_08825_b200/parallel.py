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

import os
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
    # ownership audit (parallel.py:180-188): a buffer may only hold nonzeros
    # in rows of DOFs carried by its partition's own elements -- per-row
    # flags from the device (n_dofs bytes, no nnz-sized index)
    import ctypes
    from .assembly import C_byref
    L = N.lib()
    A = ctx.new_matrix()
    dev = A._dvals.device
    st = N.stream_ptr(device=dev)
    pat = A._pattern_struct()
    flags = torch.empty(max(space.n_dofs, 1), dtype=torch.uint8, device=dev)
    for c in contexts:
        N.check(L.mf_row_touched(C_byref(pat), N.ptr(buffers[c.part]),
                                 N.ptr(flags), st), "mf_row_touched")
        touched = np.nonzero(flags[:space.n_dofs].cpu().numpy())[0]
        own = np.unique(space.element_dofs[c.owned])
        own = own[own >= 0]
        if not np.isin(touched, own).all():
            raise AssertionError("partition wrote a row outside its "
                                 "elements")
    # merge (parallel.py:190-200): every entry is the sum of the partition
    # buffers in partition order (the reference sums per row owner, which
    # gives the same per-entry order); _finish's x2 folded in
    nnz = A.nnz
    done = 0
    while done < n_parts:
        k = min(64 - (1 if done else 0), n_parts - done)
        ptrs = ([A._dvals.data_ptr()] if done else []) + [
            b.data_ptr() for b in buffers[done:done + k]]
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        last = done + k == n_parts
        N.check(L.mf_sum_ordered(len(ptrs), arr, nnz, 2.0 if last else 1.0,
                                 N.ptr(A._dvals), st), "mf_sum_ordered")
        done += k
    for c in contexts:
        c.t_t = time.perf_counter() - t_start
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
        if isinstance(weights, str) and weights == "pairs":
            # per-element candidate-pair counts (the GPU count pass): slabs
            # balanced by pair work, not by layer count
            weights = pair_counts(mesh, kernel, self.ctx.dmesh)
        self.weights = weights
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

    # -- host result without a rank-0 funnel ------------------------------
    def owned_view(self):
        """(device tensor of this rank's owned values, their offset)."""
        base = self.plan.vals_touch[0]
        a, b = self.plan.vals_own
        return self.local[a - base:b - base], a

    def copy_owned_to_host(self, host, event=None):
        """D2H of the owned row block straight into host[vals_own] (one
        slice of a node-shared array): pinned staging ring, thread-pool
        copies (device.HostStager)."""
        import torch
        from .device import HostStager
        src, a = self.owned_view()
        if src.numel() == 0:
            return
        if event is None:
            event = torch.cuda.Event()
            event.record(torch.cuda.current_stream(self.ctx.device))
        HostStager(self.ctx.device).run(src, host[a:a + src.numel()],
                                        [(event, 0, src.numel())])

    def asymmetry(self, group=None):
        """presym_asymmetry of the distributed matrix: every rank takes the
        max over its owned rows of sum_c |A_rc - A_cr| from a halo window
        (its rows plus K grid planes either side, from the owners over
        P2P), then one all-reduce MAX."""
        import torch
        import torch.distributed as dist
        from .assembly import C_byref
        win, wa = halo_window(self.local, self.plan, self.plans, self.A,
                              group)
        out = torch.zeros(1, dtype=torch.float64, device=self.ctx.device)
        r0, r1 = self.plan.rows_own
        import ctypes
        N.check(N.lib().mf_asymmetry_inf_rows(
            C_byref(self.A._pattern_struct()),
            ctypes.c_void_p(win.data_ptr() - 8 * wa), r0, r1, N.ptr(out),
            N.stream_ptr(device=self.ctx.device)), "mf_asymmetry_inf_rows")
        if self.world > 1:
            dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
        return float(out.item())


def window_range(plan, plans, A):
    """Value range [wa, wb) of the rows within K grid planes of a rank's
    owned rows (what the transposed lookups of its rows touch)."""
    K = A.K
    nplanes = A.NZ if A.NZ > 1 else A.NY
    lo_p = max(plan.own_planes[0] - K, 0)
    hi_p = min(plan.own_planes[1] + K, nplanes)
    return int(A.rowptr[lo_p * plan.plane]), int(A.rowptr[hi_p * plan.plane])


def halo_window(local, plan, plans, A, group=None):
    """This rank's owned values plus the owned values of the other ranks
    within its window_range, as one tensor (and its offset).  Every rank
    sends the part of its owned block each other rank's window needs and
    receives its own window's parts, in one batched P2P round."""
    import torch.distributed as dist
    base = plan.vals_touch[0]
    wa, wb = window_range(plan, plans, A)
    win = local.new_empty(wb - wa)
    oa, ob = plan.vals_own
    win[oa - wa:ob - wa] = local[oa - base:ob - base]
    ops = []
    for q in plans:
        if q.rank == plan.rank:
            continue
        a, b = max(q.vals_own[0], wa), min(q.vals_own[1], wb)
        if a < b:
            ops.append(dist.P2POp(dist.irecv, win[a - wa:b - wa], q.rank,
                                  group))
        qa, qb = window_range(q, plans, A)
        a, b = max(oa, qa), min(ob, qb)
        if a < b:
            ops.append(dist.P2POp(dist.isend,
                                  local[a - base:b - base].contiguous(),
                                  q.rank, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return win, wa


class SharedHostArray:
    """float64[n] backed by one file mapped by every rank of the node
    (/dev/shm when it has room, else the temp directory): each rank writes
    its own slice, rank `dst` keeps the whole array as its result."""

    def __init__(self, n, group=None, dst=0):
        import tempfile
        import torch.distributed as dist
        rank = dist.get_rank(group)
        src = dst if group is None else dist.get_global_rank(group, dst)
        name = [None]
        if rank == dst:
            d = "/dev/shm"
            try:
                st = os.statvfs(d)
                if st.f_bavail * st.f_frsize < 8 * n * 1.05:
                    d = None
            except OSError:
                d = None
            fd, path = tempfile.mkstemp(prefix="mf_vals_", dir=d)
            os.ftruncate(fd, max(8 * n, 8))
            os.close(fd)
            name = [path]
        dist.broadcast_object_list(name, src=src, group=group)
        self.path = name[0]
        self.array = np.memmap(self.path, dtype=np.float64, mode="r+",
                               shape=(max(n, 1),))[:n]
        dist.barrier(group)
        if rank == dst:
            os.unlink(self.path)     # the mappings stay valid


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


def emulate_distributed(mesh, space, kernel, config, world, device=None):
    """The host-gather path of assemble_distributed for `world` ranks, run
    rank after rank on ONE device (ranks never wait on one another): each
    rank's slab assembly, the interface additions, each rank's D2H of its
    owned block into its slice of one host array, and each rank's halo
    asymmetry over its owned rows.  Returns (host values, events,
    presym_asymmetry, per-rank timings in seconds)."""
    import ctypes

    import torch

    from .assembly import C_byref
    ranks = [SlabAssembler(mesh, space, kernel, config, r, world, device,
                           weights="pairs") for r in range(world)]
    dev = ranks[0].ctx.device
    host = np.empty(ranks[0].A.nnz, dtype=np.float64)
    timing = []
    events = 0
    for s in ranks:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        events += int(s.assemble_local()[0].item())
        torch.cuda.synchronize(dev)
        timing.append({"rank": s.rank, "assemble_s": time.perf_counter() - t0,
                       "layers": list(s.plan.layers)})
    for r in range(world - 1):           # rank r's shared top plane -> r+1
        src, dst = ranks[r], ranks[r + 1]
        a, b = src.plan.send_range
        dst.local[a - dst.plan.vals_touch[0]:b - dst.plan.vals_touch[0]] += \
            src.local[a - src.plan.vals_touch[0]:b - src.plan.vals_touch[0]]
    for s, t in zip(ranks, timing):
        t0 = time.perf_counter()
        s.copy_owned_to_host(host)
        t["d2h_s"] = time.perf_counter() - t0
        t["d2h_bytes"] = 8 * (s.plan.vals_own[1] - s.plan.vals_own[0])
    # halo windows from the merged owned blocks (what the P2P round gives)
    full = torch.empty(ranks[0].A.nnz, dtype=torch.float64, device=dev)
    for s in ranks:
        v, a = s.owned_view()
        full[a:a + v.numel()] = v
    asym = 0.0
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    for s in ranks:
        wa, wb = window_range(s.plan, s.plans, s.A)
        win = full[wa:wb].clone()
        r0, r1 = s.plan.rows_own
        N.check(N.lib().mf_asymmetry_inf_rows(
            C_byref(s.A._pattern_struct()),
            ctypes.c_void_p(win.data_ptr() - 8 * wa), r0, r1, N.ptr(out),
            N.stream_ptr(device=dev)), "mf_asymmetry_inf_rows")
        asym = max(asym, float(out.item()))
    return host, events, asym, timing


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
        N.stream_ptr(device=dev)), "mf_count_candidates")
    return counts.cpu().numpy()


def assemble_distributed(mesh, space, kernel, config=None, group=None,
                         dst=0, weights="pairs", gather="host",
                         return_slab=False):
    """Multi-GPU `assemble`: every rank of the process group calls it with
    the same host inputs; rank `dst` returns the full SparseMatrix (host
    values, events, presym_asymmetry), the others return None.

    weights="pairs" balances the slabs by candidate-pair counts.
    gather="host": each rank copies its owned row block straight into its
    slice of one node-shared host array (no rank-0 funnel; the copies of
    all ranks run in parallel), the asymmetry comes from per-rank halo
    windows.  gather="nccl" (also used for symmetrize=True): NCCL row-block
    gather to rank dst, then the single-device finish and D2H.
    return_slab=True also returns this rank's SlabAssembler (for
    assemble_rhs_distributed)."""
    import torch
    import torch.distributed as dist

    from .assembly import _d2h, check_counters
    config = config or AssemblyConfig()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    s = SlabAssembler(mesh, space, kernel, config, rank, world, dev,
                      weights=weights)
    if gather == "nccl" or config.symmetrize:
        cnt = s.assemble_local().clone()
        s.exchange(group)
        full = s.gather(group, dst)
        dist.all_reduce(cnt, group=group)
        A = None
        if rank == dst:
            A = s.A
            A._dvals = full      # the slab kernels already fold _finish's x2
            s.ctx.finish(A, cnt)
            A._vals = _d2h(A._dvals)
        return (A, s) if return_slab else A
    shm = SharedHostArray(s.A.nnz, group, dst)
    cnt = s.assemble_local().clone()
    s.exchange(group)
    s.copy_owned_to_host(shm.array)
    asym = s.asymmetry(group)
    dist.all_reduce(cnt, group=group)
    dist.barrier(group)          # every slice is in the shared array
    A = None
    if rank == dst:
        A = s.A
        c = cnt.cpu().numpy()
        check_counters(c)
        A.counters = c
        A.events = int(c[N.CNT_EVENTS])
        A.presym_asymmetry = asym
        A._vals = shm.array
    return (A, s) if return_slab else A


def assemble_rhs_distributed(mesh, space, kernel, f, g, slab, group=None,
                             dst=0):
    """`assemble_rhs` (assembly.py:679-691) over the slab decomposition:
    each rank integrates the load of its own slab elements and the matvec
    A g of its owned rows; the partial vectors (n_dofs each) are gathered
    on rank `dst` and summed there in rank order (deterministic).  Rank
    dst returns rhs[free], the others None."""
    import ctypes

    import torch
    import torch.distributed as dist

    from .assembly import C_byref, group_load_device
    from .device import to_device
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = slab.ctx.device
    L = N.lib()
    st = N.stream_ptr(device=dev)
    n = space.n_dofs
    omega = np.zeros(mesh.n_elements, dtype=bool)
    omega[mesh.omega_element_ids()] = True
    own = slab.inner[omega[slab.inner]]
    part = group_load_device(mesh, space, f, own, slab.ctx.dmesh)
    gt = np.zeros(n)
    if callable(g):
        gt[space.constrained] = g(space.dof_coords[space.constrained])
    else:
        gv = np.asarray(g, dtype=float)
        gt[space.constrained] = (gv[space.constrained]
                                 if gv.shape == (n,) else gv)
    gtd = to_device(gt, dev)
    y = torch.zeros(n, dtype=torch.float64, device=dev)
    r0, r1 = slab.plan.rows_own
    base = slab.plan.vals_touch[0]
    N.check(L.mf_matvec_rows(
        C_byref(slab.A._pattern_struct()),
        ctypes.c_void_p(slab.local.data_ptr() - 8 * base), N.ptr(gtd), r0,
        r1, N.ptr(y), st), "mf_matvec_rows")
    # partial = load part - (A g) on owned rows
    N.check(L.mf_axpby(n, 1.0, N.ptr(part), -1.0, N.ptr(y), N.ptr(part), st),
            "mf_axpby")
    if rank != dst:
        dist.send(part, dst, group)
        return None
    parts = []
    for q in range(world):
        if q == rank:
            parts.append(part)
        else:
            t = torch.empty_like(part)
            dist.recv(t, q, group)
            parts.append(t)
    tot = torch.empty_like(part)
    arr = (ctypes.c_void_p * world)(*[t.data_ptr() for t in parts])
    N.check(L.mf_sum_ordered(world, arr, n, 1.0, N.ptr(tot), st),
            "mf_sum_ordered")
    free = np.asarray(space.free, dtype=np.int64)
    fd = to_device(free, dev)
    out = torch.empty(len(free), dtype=torch.float64, device=dev)
    N.check(L.mf_gather_diff(len(free), N.ptr(fd), N.ptr(tot), None,
                             N.ptr(out), st), "mf_gather_diff")
    return out.cpu().numpy()
