"""Device-resident inputs of the assembly kernels.

`DeviceMesh` holds the mesh SoA + DOF map (mesh.py:78-88, fe_space.py:131)
in HBM and the MfMesh descriptor pointing at it; `DeviceRules` the rule
and shape tables (assembly.py:333-356); `ColorPlan` the colour-grouped
inner-element list that makes the scatter race-free: elements whose cells
have the same (x, y, z) parity and the same triangle proto share no DOF
(a DOF of cell c lies in [degree*c, degree*(c+1)] per axis), so each
colour is one atomic-free launch.
"""

import threading

import numpy as np

from . import _native as N


def _dev(device):
    import torch
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def to_device(arr, device, pinned=True):
    """numpy -> device tensor through a pinned staging copy (device None =
    the current CUDA device)."""
    import torch
    dev = _dev(device)
    if dev.type != "cuda":
        raise ValueError(f"to_device needs a CUDA device, got {dev}")
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    t = torch.from_numpy(a)
    if pinned and t.numel() > 0:
        t = t.pin_memory()
    return t.to(dev, non_blocking=True)


def cell_ptr_of(mesh):
    """(flat cell id per element, CSR of elements per cell).

    Our meshes provide `cell_ptr()`; the reference's Mesh does not (its
    `_cell_ptr(mesh)` is a free function, assembly.py:135-148), so for any
    other mesh object the same arrays are computed here from `elem_cell`
    and `grid_ncells` (elements are cell-lex ordered, mesh.py:209-253)."""
    if hasattr(mesh, "cell_ptr"):
        return mesh.cell_ptr()
    c = np.asarray(mesh.elem_cell)
    nc = mesh.grid_ncells
    flat = c[:, 1].astype(np.int64) * nc[0] + c[:, 0]
    if mesh.dim == 3:
        flat += c[:, 2].astype(np.int64) * (nc[0] * nc[1])
    flat = flat.astype(np.int32)
    ncells = int(np.prod(nc))
    return flat, np.searchsorted(flat, np.arange(ncells + 1)).astype(np.int64)


class DeviceMesh:
    """Mesh + FE space arrays in device memory (our host layer's objects or
    the reference's Mesh/FESpace, which carry the same SoA arrays)."""

    def __init__(self, mesh, space, device=None):
        dev = _dev(device)
        self.device = dev
        self.dim = mesh.dim
        flat, cptr = cell_ptr_of(mesh)
        nc = mesh.grid_ncells
        host = {
            "elem_kind": np.ascontiguousarray(mesh.elem_kind, np.int8),
            "elem_coords": np.ascontiguousarray(mesh.elem_coords, np.float64),
            "elem_lo": np.ascontiguousarray(mesh.elem_lo, np.float64),
            "elem_hi": np.ascontiguousarray(mesh.elem_hi, np.float64),
            "elem_dofs": np.ascontiguousarray(space.element_dofs, np.int64),
            "elem_cell": np.ascontiguousarray(flat, np.int32),
            "cell_ptr": np.ascontiguousarray(cptr, np.int64),
        }
        self.h2d_bytes = sum(a.nbytes for a in host.values())
        self.t = {k: to_device(v, dev) for k, v in host.items()}
        self.struct = N.MfMesh(
            dim=mesh.dim, degree=space.degree, n_elem=mesh.n_elements,
            nv_max=mesh.elem_coords.shape[1],
            nloc_max=space.element_dofs.shape[1],
            elem_kind=self.t["elem_kind"].data_ptr(),
            elem_coords=self.t["elem_coords"].data_ptr(),
            elem_lo=self.t["elem_lo"].data_ptr(),
            elem_hi=self.t["elem_hi"].data_ptr(),
            elem_dofs=self.t["elem_dofs"].data_ptr(),
            elem_cell=self.t["elem_cell"].data_ptr(),
            cell_ptr=self.t["cell_ptr"].data_ptr(),
            ncx=int(nc[0]), ncy=int(nc[1]),
            ncz=int(nc[2]) if mesh.dim == 3 else 1,
            kinds_present=int(np.bitwise_or.reduce(
                1 << np.unique(mesh.elem_kind).astype(np.int64))),
            layout=1 if getattr(mesh, "unstructured", False) else 0,
            row_period=int(getattr(mesh, "row_period", 2)))


class DeviceRules:
    """Rule/shape tables of a `PrepTables` (or of the reference's `_Prep`,
    assembly.py:333-356) in device memory.

    The specialised box kernels sum-factorise over the 1D factors of the
    tensor rules.  `PrepTables` carries them; for the reference's `_Prep`,
    which does not, pass `box_1d=(outer_1d, inner_1d)` (e.g. from
    `assembly.rule_1d(config.outer_rule)`) or leave them out, which sends
    box meshes to the generic kernel (n1d = 0)."""

    def __init__(self, prep, device=None, box_1d=None):
        dev = _dev(device)
        names = ["box_out_pts", "box_out_w", "box_in_pts", "box_in_w",
                 "tri_out_pts", "tri_out_w", "tri_in_pts", "tri_in_w"]
        host = {n: getattr(prep, n) for n in names}
        host["phi_box_in"] = prep.PHI_box_in
        host["phi_tri_in"] = prep.PHI_tri_in
        if box_1d is None:
            box_1d = (getattr(prep, "box_out_1d", None),
                      getattr(prep, "box_in_1d", None))
        empty = (np.zeros(1), np.zeros(1))
        o1, i1 = (b if b is not None else empty for b in box_1d)
        host["box_out_x1d"], host["box_out_w1d"] = o1
        host["box_in_x1d"], host["box_in_w1d"] = i1
        n1d_out = len(o1[0]) if box_1d[0] is not None else 0
        n1d_in = len(i1[0]) if box_1d[1] is not None else 0
        self.t = {k: to_device(np.ascontiguousarray(v, np.float64), dev,
                               pinned=False) for k, v in host.items()}
        p = {k: v.data_ptr() for k, v in self.t.items()}
        self.struct = N.MfRules(
            nq_box_out=len(prep.box_out_w), nq_box_in=len(prep.box_in_w),
            nq_tri_out=len(prep.tri_out_w), nq_tri_in=len(prep.tri_in_w),
            n1d_box_out=n1d_out, n1d_box_in=n1d_in, **p)


def _nproto(mesh):
    return 6 if getattr(mesh, "kind", None) == "tet" else 2


def ncolors_of(mesh):
    """Colours of `color_of`: 16 (2 protos), 48 for Kuhn tets (6 protos),
    the greedy colour count of an unstructured mesh."""
    if getattr(mesh, "unstructured", False):
        return int(mesh.n_colors)
    return 8 * _nproto(mesh)


def color_of(mesh):
    """Colour id per element: cell parity bits * nproto + proto.

    Elements of one colour have one proto and lie in cells of one parity
    (two apart on some axis), so they share no DOF (race-free scatter).
    Unstructured meshes carry a greedy vertex-disjoint colouring."""
    if getattr(mesh, "unstructured", False):
        return np.asarray(mesh.elem_color, dtype=np.int64)
    c = mesh.elem_cell.astype(np.int64)
    col = (c[:, 0] & 1) | ((c[:, 1] & 1) << 1)
    if mesh.dim == 3:
        col |= (c[:, 2] & 1) << 2
    return (col * _nproto(mesh)
            + mesh.elem_proto.astype(np.int64)).astype(np.int64)


class ColorPlan:
    """Inner elements grouped by colour (one launch per group).

    Default: ascending ids inside a colour.  With `work` (per-element work
    estimate, e.g. candidate-pair counts) each group is ordered heaviest
    first, so the last wave of a launch holds the light elements (shorter
    tail).  With `layers` (a list of top-axis cell-layer ranges) the groups
    are (layer range, colour) in that order, so the rows of a finished
    range can leave the device while the next range computes.
    """

    NCOLORS = 16

    def __init__(self, mesh, inner_ids=None, device=None, work=None,
                 layers=None):
        col = color_of(mesh)
        self.NCOLORS = ncolors_of(mesh)
        ids = (np.arange(mesh.n_elements, dtype=np.int64) if inner_ids is None
               else np.asarray(inner_ids, dtype=np.int64))
        if layers is None:
            slab = np.zeros(len(ids), dtype=np.int64)
            nslab = 1
        else:
            layer = mesh.elem_cell[ids, mesh.dim - 1]
            cuts = np.asarray([a for a, _ in layers] + [layers[-1][1]])
            slab = np.searchsorted(cuts, layer, side="right") - 1
            nslab = len(layers)
        key2 = (np.zeros(len(ids)) if work is None
                else -np.asarray(work, dtype=np.float64)[ids])
        group = slab * self.NCOLORS + col[ids]
        order = np.lexsort((ids, key2, group))
        ids = ids[order]
        self.ngroups = nslab * self.NCOLORS
        counts = np.bincount(group[order], minlength=self.ngroups)
        self.color_ptr = np.zeros(self.ngroups + 1, dtype=np.int64)
        np.cumsum(counts, out=self.color_ptr[1:])
        self.inner_sorted = to_device(ids.astype(np.int32), _dev(device))
        self.n_inner = int(len(ids))
        self.h2d_bytes = ids.size * 4
        self.layers = layers

    def group_range(self, slab):
        """(first, last) group index of one layer range."""
        return slab * self.NCOLORS, (slab + 1) * self.NCOLORS


class HostStager:
    """Device -> fresh host array at pinned-copy speed.

    A pinned staging ring (allocated once per process and device, reused by
    every call) takes the DMA at full rate; a thread pool copies each
    staged chunk into the caller's pageable result array, which also
    spreads its first-touch page faults over the threads.  Ranges are
    enqueued with the CUDA event after which they are final, so the copies
    overlap the remaining device work.
    """

    CHUNK = 1 << 25          # doubles per staging chunk (256 MiB)
    NBUF = 4
    _rings = {}
    _locks = {}
    _guard = threading.Lock()

    def __init__(self, device, threads=16):
        import torch
        self.device = torch.device(device)
        key = str(self.device)
        with HostStager._guard:
            if key not in HostStager._rings:
                HostStager._rings[key] = [
                    torch.empty(self.CHUNK, dtype=torch.float64,
                                pin_memory=True)
                    for _ in range(self.NBUF)]
                HostStager._locks[key] = threading.Lock()
        self.ring = HostStager._rings[key]
        # one transfer at a time per device: the ring is shared by every
        # caller in the process (two concurrent copies would interleave
        # their chunks in the same staging buffers)
        self.lock = HostStager._locks[key]
        self.stream = torch.cuda.Stream(device=self.device)
        self.threads = threads

    def prefault(self, host, chunk=1 << 24):
        """Touch every page of `host` (zero fill) with the thread pool."""
        from concurrent.futures import ThreadPoolExecutor
        n = host.shape[0]

        def touch(a):
            host[a:a + chunk].fill(0.0)

        with ThreadPoolExecutor(max_workers=self.threads) as pool:
            list(pool.map(touch, range(0, n, chunk)))

    def run(self, src, host, ranges):
        """Copy src[a:b] -> host[a:b] for each (event, a, b), in order
        (serialised per device: the staging ring is shared)."""
        with self.lock:
            self._run(src, host, ranges)

    def _run(self, src, host, ranges):
        import torch
        from concurrent.futures import ThreadPoolExecutor
        import os
        import time
        trace = os.environ.get("MF_STAGER_TRACE") == "1"
        t0 = time.perf_counter()
        pending = [None] * self.NBUF     # host-copy futures per buffer
        k = 0
        with ThreadPoolExecutor(max_workers=self.threads) as pool:
            for ri, (ev, a, b) in enumerate(ranges):
                if trace:
                    tw = time.perf_counter()
                    ev.synchronize()
                    print(f"[stager] range {ri}: worker reached it at "
                          f"{tw:.3f}, event done at {time.perf_counter():.3f}"
                          f" ({(b - a) * 8 / 1e9:.2f} GB)", flush=True)
                self.stream.wait_event(ev)
                for c0 in range(a, b, self.CHUNK):
                    c1 = min(b, c0 + self.CHUNK)
                    slot = k % self.NBUF
                    if pending[slot] is not None:
                        for f in pending[slot]:
                            f.result()
                    buf = self.ring[slot][:c1 - c0]
                    with torch.cuda.stream(self.stream):
                        buf.copy_(src[c0:c1], non_blocking=True)
                    done = torch.cuda.Event()
                    done.record(self.stream)
                    dst = host[c0:c1]
                    bv = buf.numpy()
                    nsub = self.threads
                    step = -(-(c1 - c0) // nsub)

                    def piece(j, done=done, dst=dst, bv=bv, step=step):
                        done.synchronize()
                        np.copyto(dst[j * step:(j + 1) * step],
                                  bv[j * step:(j + 1) * step])

                    pending[slot] = [pool.submit(piece, j)
                                     for j in range(nsub)]
                    k += 1
            for fl in pending:
                if fl is not None:
                    for f in fl:
                        f.result()
        if trace:
            print(f"[stager] started {t0:.3f}, all copies done at "
                  f"{time.perf_counter():.3f}", flush=True)
