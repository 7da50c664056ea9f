"""Stiffness/load assembly entry points (reference rows a4-a14, boundary 8(b)).

Host orchestration for the B200 path.  Mirrors the reference module
`mollifem/assembly.py` -- same names, arguments, return contract and
ValueError behaviour -- while every numeric kernel on the path runs in
`csrc/` through the C-ABI in `include/mollifem_b200.h`:

  assemble()            assembly.py:456-473  -> mf_general_core (+ mf_scale
                                                 folded, mf_asymmetry_inf)
  neighbor_sets()       assembly.py:178-183  -> mf_count/fill_candidates
  assemble_rhs()        assembly.py:679-691  -> mf_load_scatter, mf_matvec
  SparseMatrix methods  assembly.py:189-310  -> mf_matvec/diag/...

The matrix is A = 2(A21 + A22) on the implicit structured pattern (row r
couples to the clipped grid box of half-width K around r).  There is no
CPU fallback: without the CUDA library every device call raises.
"""

import math
import os

import numpy as np

from .fe_space import eval_shape_functions
from .kernel import mollifier  # noqa: F401  (re-exported like the reference)
from .mesh import BoundingBox
from .quadrature import rule_for_kind

__all__ = ["AssemblyConfig", "SparseMatrix", "NeighborSets", "assemble",
           "assemble_rhs", "neighbor_sets", "pattern_halfwidth",
           "aprx_min_dist", "aprx_max_dist"]


class AssemblyConfig:
    """Method, recursion window [L_min, L_max], rule presets, strategy.

    Validation follows assembly.py:58-78; strategies as in the reference
    ("auto" = blocked on pure meshes, general otherwise).
    """

    def __init__(self, method="mollified_adaptive", L_min=1, L_max=3,
                 outer_rule="default", inner_rule="default", strategy="auto",
                 symmetrize=False):
        if method not in ("mollified_adaptive", "barycenter"):
            raise ValueError(f"unknown assembly method {method!r}")
        if not 1 <= L_min <= L_max:
            raise ValueError("need 1 <= L_min <= L_max")
        if L_max > 24:
            raise ValueError("L_max > 24 exceeds the recursion stack bound")
        if strategy not in ("auto", "general", "blocked"):
            raise ValueError(f"unknown strategy {strategy!r}")
        self.method = method
        self.L_min = int(L_min)
        self.L_max = int(L_max)
        self.outer_rule = outer_rule
        self.inner_rule = inner_rule
        self.strategy = strategy
        self.symmetrize = bool(symmetrize)

    def __repr__(self):
        return (f"AssemblyConfig({self.method}, L=[{self.L_min},"
                f"{self.L_max}], outer={self.outer_rule!r}, "
                f"inner={self.inner_rule!r}, strategy={self.strategy})")


# ---------------------------------------------------------------------------
# conservative box distances (assembly.py:96-111)

def _box_lo_hi(box):
    if isinstance(box, BoundingBox):
        return box.lo, box.hi
    lo, hi = box
    return np.asarray(lo, dtype=float), np.asarray(hi, dtype=float)


def aprx_min_dist(box_a, box_b):
    """Largest single-axis gap (0 if the boxes overlap): a lower bound."""
    alo, ahi = _box_lo_hi(box_a)
    blo, bhi = _box_lo_hi(box_b)
    return float(max(np.maximum(alo - bhi, blo - ahi).max(), 0.0))


def aprx_max_dist(box_a, box_b):
    """Euclidean norm of per-axis extreme separations: an upper bound."""
    alo, ahi = _box_lo_hi(box_a)
    blo, bhi = _box_lo_hi(box_b)
    d = np.maximum(np.abs(alo - bhi), np.abs(blo - ahi))
    return float(np.sqrt((d * d).sum()))


def stencil_radius(reach, h):
    """Cell stencil radius R = floor(reach/h + 1e-12) + 1 (assembly.py:151)."""
    return int(math.floor(reach / h + 1e-12)) + 1


def stencil_pad(mesh):
    """Extra stencil reach for meshes whose element boxes leave their cells
    (jittered tets; 0 for the reference's structured meshes)."""
    return float(getattr(mesh, "stencil_pad", 0.0))


def pattern_halfwidth(mesh, params, config, degree):
    """(K, oe): grid half-width of a row's coupling box (assembly.py:313)."""
    if config.method == "barycenter":
        f = 2.0 / 3.0 if mesh.kind in ("tri", "mixed") else 0.5
        oe = int(math.floor(params.delta / mesh.h + f + 1e-12))
    else:
        # unstructured meshes: coupled vertices may sit further apart in
        # lattice index than their elements' bins (mesh.DelaunayMesh)
        pad = float(getattr(mesh, "pattern_pad", stencil_pad(mesh)))
        oe = int(math.floor((params.delta + params.eps + pad)
                            / mesh.h + 1e-12)) + 1
    return degree * (oe + 1), oe


# ---------------------------------------------------------------------------
# rule / table preparation (assembly.py:333-356)

class PrepTables:
    """Outer/inner reference rules and inner shape tables for one config."""

    def __init__(self, mesh, space, config):
        dim = mesh.dim
        box_kind = "hex" if dim == 3 else "quad"
        outer = config.outer_rule
        inner = config.inner_rule
        if outer == "default" and config.method == "barycenter":
            outer = "lobatto3"
        # simplex slots ("tri_*"): triangles in 2D, tetrahedra in 3D (the
        # tet element is new; its rules are "default" = tet4, tet1/4/11)
        simplex = "tet" if mesh.kind == "tet" else "tri"
        tri_presets = ("tri3", "tri6", "tri7")
        tri_preset = outer in tri_presets or inner in tri_presets
        if tri_preset and mesh.kind != "tri":
            raise ValueError("tri3/tri6/tri7 presets need a pure triangle "
                             "mesh")
        if simplex == "tet" or tri_preset:
            box_outer = box_inner = "gauss2"   # unused placeholders
        else:
            box_outer, box_inner = outer, inner
        self.box_out = rule_for_kind(box_kind, box_outer)
        self.box_in = rule_for_kind(box_kind, box_inner)
        self.tri_out = rule_for_kind(simplex, outer)
        self.tri_in = rule_for_kind(simplex, inner)
        deg = space.degree
        self.PHI_box_in = np.ascontiguousarray(
            eval_shape_functions(box_kind, deg, self.box_in.ref_points))
        self.PHI_tri_in = np.ascontiguousarray(
            eval_shape_functions(simplex, deg, self.tri_in.ref_points))
        self.box_out_pts = np.ascontiguousarray(self.box_out.ref_points)
        self.box_out_w = np.ascontiguousarray(self.box_out.weights)
        self.box_in_pts = np.ascontiguousarray(self.box_in.ref_points)
        self.box_in_w = np.ascontiguousarray(self.box_in.weights)
        self.tri_out_pts = np.ascontiguousarray(self.tri_out.ref_points)
        self.tri_out_w = np.ascontiguousarray(self.tri_out.weights)
        self.tri_in_pts = np.ascontiguousarray(self.tri_in.ref_points)
        self.tri_in_w = np.ascontiguousarray(self.tri_in.weights)
        # 1D factors of the tensor box rules (for sum factorisation)
        self.box_out_1d = _rule_1d(box_outer)
        self.box_in_1d = _rule_1d(box_inner)


def rule_1d(preset):
    """(1D points on [-1, 1], weights) of a tensor box rule preset."""
    return _rule_1d(preset)


def _rule_1d(preset):
    from .quadrature import _preset, gauss_legendre_1d, gauss_lobatto_1d
    fam, n = _preset(preset)
    r = gauss_legendre_1d(n) if fam == "gauss" else gauss_lobatto_1d(n)
    return (np.ascontiguousarray(r.ref_points[:, 0]),
            np.ascontiguousarray(r.weights))


def prep_tables(mesh, space, config):
    return PrepTables(mesh, space, config)


# ---------------------------------------------------------------------------
# implicit-pattern matrix

class HostPattern:
    """Pattern metadata + a host value array (assembly.py:197-223)."""

    def _init_pattern(self, space, K):
        dims = space.grid_dims
        self.NX = int(dims[0])
        self.NY = int(dims[1])
        self.NZ = int(dims[2]) if len(dims) == 3 else 1
        self.K = int(K)
        self.n = int(space.n_dofs)
        r = np.arange(self.n, dtype=np.int64)
        self.gx = (r % self.NX).astype(np.int32)
        t = r // self.NX
        self.gy = (t % self.NY).astype(np.int32)
        self.gz = (t // self.NY).astype(np.int32)

        def width(g, N):
            lo = np.maximum(g - self.K, 0)
            hi = np.minimum(g + self.K, N - 1)
            return (hi - lo + 1).astype(np.int64)

        row_nnz = width(self.gx, self.NX) * width(self.gy, self.NY)
        if self.NZ > 1:
            row_nnz *= width(self.gz, self.NZ)
        self.rowptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(row_nnz, out=self.rowptr[1:])
        self.presym_asymmetry = None
        self.events = None

    def __init__(self, space, K, allocate=True):
        self._init_pattern(space, K)
        self._vals = (np.zeros(int(self.rowptr[-1]), dtype=np.float64)
                      if allocate else None)

    @classmethod
    def for_space(cls, mesh, space, params, config):
        K, oe = pattern_halfwidth(mesh, params, config, space.degree)
        A = cls(space, K)
        A._offset_reach = oe
        return A

    @property
    def vals(self):
        return self._vals

    @vals.setter
    def vals(self, v):
        self._vals = v

    @property
    def nnz(self):
        return int(self.rowptr[-1])

    @property
    def n_rows(self):
        return self.n

    @property
    def n_cols(self):
        return self.n

    @property
    def shape(self):
        return (self.n, self.n)

    def row_cols(self, r):
        xlo = max(self.gx[r] - self.K, 0)
        xhi = min(self.gx[r] + self.K, self.NX - 1)
        ylo = max(self.gy[r] - self.K, 0)
        yhi = min(self.gy[r] + self.K, self.NY - 1)
        zlo = max(self.gz[r] - self.K, 0)
        zhi = min(self.gz[r] + self.K, self.NZ - 1)
        cx = np.arange(xlo, xhi + 1)
        cy = np.arange(ylo, yhi + 1)
        cz = np.arange(zlo, zhi + 1)
        return ((cz[:, None, None] * self.NY + cy[None, :, None]) * self.NX
                + cx[None, None, :]).ravel()

    def row_entries(self, r):
        return self.row_cols(r), self.vals[self.rowptr[r]:self.rowptr[r + 1]]

    def __repr__(self):
        return f"{type(self).__name__}(n={self.n}, K={self.K}, nnz={self.nnz})"


class SparseMatrix(HostPattern):
    """Values-only matrix on the structured DOF grid (assembly.py:189-310).

    After `assemble()` the values live in HBM (`vals_device`) and, unless
    the caller asked for a device-only result, in the host array `vals`
    (the reference contract).  Every method runs on the device through the
    C-ABI.  While a device copy exists the host array is READ-ONLY, so an
    in-place edit cannot leave the device copy silently stale: to change
    values assign a new array (`A.vals = v`, which drops the device copy;
    the next device method uploads it).  Matrices without a device copy
    (`copy_pattern()`) have a writable `vals`, as in the reference.
    """

    def __init__(self, space, K, allocate=True):
        super().__init__(space, K, allocate=allocate)
        self._dvals = None
        self._drowptr = None
        self.counters = None

    # -- device plumbing -------------------------------------------------
    def _pattern_struct(self):
        from . import _native as N
        if self._drowptr is None:
            from .device import to_device
            self._drowptr = to_device(
                self.rowptr,
                self._dvals.device if self._dvals is not None else None)
        return N.MfPattern(NX=self.NX, NY=self.NY, NZ=self.NZ, K=self.K,
                           n=self.n, rowptr=self._drowptr.data_ptr())

    @property
    def vals_device(self):
        if self._dvals is None:
            self.sync_to_device()
        return self._dvals

    def sync_to_device(self, device=None):
        from .device import to_device
        if self._vals is None:
            raise RuntimeError("matrix has no values")
        self._dvals = to_device(self._vals, device)
        _freeze(self._vals)
        return self._dvals

    @property
    def vals(self):
        if self._vals is None and self._dvals is not None:
            self._vals = _d2h(self._dvals)
        if self._dvals is not None:
            _freeze(self._vals)
        return self._vals

    @vals.setter
    def vals(self, v):
        self._vals = v
        self._dvals = None

    def _call(self, name, *args):
        from . import _native as N
        L = N.lib()
        N.check(getattr(L, name)(C_byref(self._pattern_struct()), *args,
                                 N.stream_ptr(device=self._dvals.device)),
                name)

    def _dev_vec(self, x):
        import torch
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"vector length must be {self.n}")
        return torch.from_numpy(x).to(self.vals_device.device)

    # -- reference methods -------------------------------------------------
    def matvec(self, x):
        import torch
        from . import _native as N
        xd = self._dev_vec(x)
        yd = torch.empty_like(xd)
        self._call("mf_matvec", N.ptr(self.vals_device), N.ptr(xd),
                   N.ptr(yd))
        return yd.cpu().numpy()

    def __matmul__(self, x):
        return self.matvec(x)

    def symmetrize_(self):
        from . import _native as N
        self._call("mf_symmetrize", N.ptr(self.vals_device))
        self._vals = None  # host copy refreshed lazily from the device

    def _reduce(self, name):
        import torch
        from . import _native as N
        out = torch.zeros(1, dtype=torch.float64,
                          device=self.vals_device.device)
        self._call(name, N.ptr(self.vals_device), N.ptr(out))
        return float(out.item())

    def asymmetry_inf(self):
        """inf-norm of A - A^T."""
        return self._reduce("mf_asymmetry_inf")

    def norm_inf(self):
        return self._reduce("mf_norm_inf")

    def diag(self):
        import torch
        from . import _native as N
        out = torch.empty(self.n, dtype=torch.float64,
                          device=self.vals_device.device)
        self._call("mf_diag", N.ptr(self.vals_device), N.ptr(out))
        return out.cpu().numpy()

    def to_scipy(self):
        import torch
        from scipy.sparse import csr_matrix
        from . import _native as N
        cols = torch.empty(self.nnz, dtype=torch.int64,
                           device=self.vals_device.device)
        self._call("mf_fill_cols", N.ptr(cols))
        return csr_matrix((self.vals.copy(), cols.cpu().numpy(),
                           self.rowptr.copy()), shape=(self.n, self.n))

    def toarray(self):
        return self.to_scipy().toarray()

    def copy_pattern(self):
        """All-zero host matrix sharing this pattern's metadata."""
        other = object.__new__(SparseMatrix)
        for a in ("NX", "NY", "NZ", "K", "n", "gx", "gy", "gz", "rowptr"):
            setattr(other, a, getattr(self, a))
        other._vals = np.zeros(self.nnz)
        other._dvals = None
        other._drowptr = self._drowptr
        other.presym_asymmetry = None
        other.events = None
        other.counters = None
        return other


def _freeze(a):
    """Host values mirrored on the device are read-only (SparseMatrix)."""
    if isinstance(a, np.ndarray) and a.flags.writeable:
        try:
            a.setflags(write=False)
        except ValueError:
            pass


def C_byref(s):
    import ctypes
    return ctypes.byref(s)


# below this many value bytes a matrix is copied to the host in one plain
# transfer after the kernels (no staging ring, no overlapped ranges)
_STREAM_MIN_BYTES = 1 << 28


def _d2h(t):
    """Device float64 vector -> fresh host numpy array (HostStager for
    large arrays, a plain copy below _STREAM_MIN_BYTES)."""
    import torch
    from .device import HostStager
    if t.numel() == 0:
        return np.zeros(0, dtype=np.float64)
    if (t.dtype != torch.float64 or t.dim() != 1
            or t.numel() * 8 < _STREAM_MIN_BYTES):
        return t.cpu().numpy()
    host = np.empty(t.numel(), dtype=np.float64)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(t.device))
    HostStager(t.device).run(t, host, [(ev, 0, t.numel())])
    return host


def _new_matrix(mesh, space, params, config, allocate):
    K, oe = pattern_halfwidth(mesh, params, config, space.degree)
    A = SparseMatrix(space, K, allocate=allocate)
    A._offset_reach = oe
    return A


# ---------------------------------------------------------------------------
# neighbour sets (assembly.py:117-183)

class NeighborSets:
    """CSR candidate lists: inner m of outer l with box gap < delta+eps."""

    def __init__(self, outer_ids, ptr, ids):
        self.outer_ids = outer_ids
        self.ptr = ptr
        self.ids = ids
        self._pos = {int(l): i for i, l in enumerate(outer_ids)}

    def of(self, l):
        i = self._pos[int(l)]
        return self.ids[self.ptr[i]:self.ptr[i + 1]]

    def __len__(self):
        return len(self.outer_ids)


def candidates(mesh, reach, outer_ids, inner_mask, device=None,
               dmesh=None, return_device=False):
    """(ptr, ids) of `_candidates` (assembly.py:157-175), computed on GPU."""
    import torch
    from . import _native as N
    from .device import DeviceMesh, to_device
    L = N.lib()
    if dmesh is None:
        dmesh = DeviceMesh(mesh, _DummySpace(mesh), device)
    dev = dmesh.device
    outer = to_device(np.ascontiguousarray(outer_ids, np.int64), dev)
    mask = to_device(np.ascontiguousarray(inner_mask, np.uint8), dev)
    n = int(outer.numel())
    R = stencil_radius(reach + stencil_pad(mesh), mesh.h)
    st = N.stream_ptr(device=dev)
    counts = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    N.check(L.mf_count_candidates(C_byref(dmesh.struct), N.ptr(outer), n,
                                  N.ptr(mask), R, float(reach), N.ptr(counts),
                                  st), "mf_count_candidates")
    ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    wsb = int(L.mf_scan_workspace_bytes(n))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    N.check(L.mf_exclusive_scan(N.ptr(counts), n, N.ptr(ptr), N.ptr(ws), wsb,
                                st), "mf_exclusive_scan")
    total = int(ptr[-1].item())
    ids = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    N.check(L.mf_fill_candidates(C_byref(dmesh.struct), N.ptr(outer), n,
                                 N.ptr(mask), R, float(reach), N.ptr(ptr),
                                 N.ptr(ids), st), "mf_fill_candidates")
    ids = ids[:total]
    if return_device:
        return ptr, ids
    return ptr.cpu().numpy(), ids.cpu().numpy()


class _DummySpace:
    """Degree-1 stand-in when only geometry is needed on the device."""

    def __init__(self, mesh):
        self.degree = 1
        self.element_dofs = np.zeros((mesh.n_elements, 1), dtype=np.int64)


def neighbor_sets(mesh, params):
    """Candidate inner elements per outer element for kernel params."""
    outer = np.arange(mesh.n_elements, dtype=np.int64)
    mask = np.ones(mesh.n_elements, dtype=np.uint8)
    ptr, ids = candidates(mesh, params.delta + params.eps, outer, mask)
    return NeighborSets(outer, ptr, ids)


# ---------------------------------------------------------------------------
# assembly

class AssemblyContext:
    """Device-resident inputs of one (mesh, space, kernel, config) problem.

    `assemble()` builds one per call (inputs copied host->device inside
    the call, as the end-to-end contract requires); benchmarks and the
    partitioned driver may build it once and call `run()` repeatedly.
    """

    def __init__(self, mesh, space, params, config, device=None):
        from .device import DeviceMesh, DeviceRules
        self.mesh, self.space, self.params, self.config = (mesh, space,
                                                           params, config)
        self.prep = prep_tables(mesh, space, config)
        self.dmesh = DeviceMesh(mesh, space, device)
        self.drules = DeviceRules(self.prep, device)
        self.device = self.dmesh.device
        self.R = stencil_radius(params.delta + params.eps + stencil_pad(mesh),
                                mesh.h)
        self.h2d_bytes = self.dmesh.h2d_bytes

    def default_plan(self):
        """All elements, colour groups ordered heaviest first (candidate
        pair counts from the GPU count pass)."""
        from .device import ColorPlan
        from .parallel import pair_counts
        if getattr(self, "_plan", None) is None:
            work = pair_counts(self.mesh, self.params, self.dmesh)
            self._plan = ColorPlan(self.mesh, None, self.device, work=work)
        return self._plan

    def kernel_struct(self):
        from . import _native as N
        p, c = self.params, self.config
        return N.MfKernel(delta=p.delta, eps=p.eps, cde=p.c_delta_eps,
                          L_min=c.L_min, L_max=c.L_max)

    def new_matrix(self):
        import torch
        A = _new_matrix(self.mesh, self.space, self.params, self.config,
                        allocate=False)
        A._dvals = torch.zeros(A.nnz, dtype=torch.float64, device=self.device)
        from .device import to_device
        A._drowptr = to_device(A.rowptr, self.device)
        self.h2d_bytes += A.rowptr.nbytes
        return A

    def run(self, A, outer_mask=None, inner_ids=None, scale=2.0, flags=0,
            plan=None, counters=None, vals_window=None, groups=None):
        """Accumulate scale*(A21 + A22) of the selected pairs into A.

        vals_window: a `WindowedValues` when the caller only holds the
        value range of the rows its inner elements touch (multi-GPU)."""
        import torch
        from . import _native as N
        from .device import ColorPlan, to_device
        L = N.lib()
        n = self.mesh.n_elements
        if outer_mask is None:
            om = torch.ones(n, dtype=torch.uint8, device=self.device)
        else:
            om = to_device(np.ascontiguousarray(outer_mask, np.uint8),
                           self.device)
        if plan is None:
            plan = (self.default_plan() if inner_ids is None and
                    outer_mask is None else
                    ColorPlan(self.mesh, inner_ids, self.device))
        if counters is None:
            counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64,
                                   device=self.device)
        wsb = int(L.mf_general_workspace_bytes(C_byref(self.dmesh.struct),
                                               C_byref(self.drules.struct),
                                               plan.n_inner))
        ws = torch.zeros(wsb, dtype=torch.uint8, device=self.device)
        g0, g1 = groups if groups is not None else (0, plan.ngroups)
        cptr = np.ascontiguousarray(plan.color_ptr[g0:g1 + 1])
        cp = cptr.ctypes.data_as(ctypes_void_p())
        N.check(L.mf_general_core(
            C_byref(self.dmesh.struct), C_byref(self.drules.struct),
            C_byref(self.kernel_struct()), C_byref(A._pattern_struct()),
            N.ptr(om), N.ptr(plan.inner_sorted), cp, g1 - g0, self.R,
            float(scale),
            (vals_window.pointer() if vals_window is not None
             else N.ptr(A._dvals)), N.ptr(counters), int(flags),
            N.ptr(ws), wsb, N.stream_ptr(device=self.device)), "mf_general_core")
        return counters

    # -- general path with the host copy overlapped -----------------------
    def run_streamed(self, A, flags=0, nslabs=None, strategy="general"):
        """General path in top-axis layer ranges: while range s+1 computes,
        the rows finished by range s (their DOF planes are touched by no
        later layer) are copied device->host on a side stream by a worker
        thread into the result array.  Same kernels and launches otherwise;
        call `finish` then `join_streamed`."""
        import threading

        import torch
        from . import _native as N
        from .device import ColorPlan, HostStager
        from .parallel import pair_counts, slab_layers, slab_layers_fracs
        mesh, space = self.mesh, self.space
        axis = mesh.dim - 1
        nl = int(mesh.grid_ncells[axis])
        gather = strategy == "blocked" and space.degree == 1
        fr = os.environ.get("MF_STREAM_FRACS")
        if gather:
            # The entry-wise gather writes whole rows, has no colours (no
            # launch tails) and runs about as long as the copy of what it
            # writes, so it streams in many even ranges: the copy of range
            # s overlaps the gather of range s+1 (R4 default path, host in
            # to host out: 0.82 s with the general path's [0.9, 1] cut,
            # which copied 90% of the matrix after computing it).  No pair
            # counts and no colour plan are needed here.
            work = None
            if fr:
                fracs = [float(x) for x in fr.split(",")]
            else:
                n = 8 if A.nnz * 8 > 2**30 else (2 if A.nnz * 8 > 2**28
                                                  else 1)
                fracs = [(k + 1) / n for k in range(n)]
            fracs = fracs[-max(1, min(len(fracs), nl // 4)):]
            fracs[-1] = 1.0
            layers = slab_layers_fracs(mesh, fracs, None)
            plan = None
        else:
            work = pair_counts(mesh, self.params, self.dmesh)
            if nslabs is not None:
                layers = slab_layers(mesh, nslabs, work)
            else:
                # few ranges (every range adds a launch tail per colour),
                # the last one small (its copy is exposed).
                # cuts are fractions of the top-axis LAYERS (rows), not of
                # the pair work: the time per pair varies across the
                # domain, and what must be small is the byte count of the
                # ranges that finish last (traced on R4: work-based cuts
                # left 6.5 GB to copy after the kernels)
                # With the copies running during the kernels (finish waits
                # on an event), two ranges suffice.  Measured end to end:
                # R4 (16 GB) 7.96 s with [0.5, 0.8, 0.93, 1] -> 7.78 s with
                # [0.9, 1]; R3-16h (3.2 GB) 0.90 s with [0.5, 1], 1.12 s
                # with [0.75, 1], 1.18 s with [0.9, 1] (its
                # thread-per-element launches pay a long per-thread tail on
                # a thin range); R2 is indifferent (1.55 s).
                if fr:
                    fracs = [float(x) for x in fr.split(",")]
                elif A.nnz * 8 > 2**33:
                    # k_hex2 runs one warp per block, so a range's launch
                    # tails are short now: R4 e2e 4.652 s with [0.9, 1],
                    # 4.615 s with these four, 4.86 s with [0.95, 1]
                    # (the thread-level kernels keep two ranges: every
                    # range costs them a tail per colour launch)
                    fracs = ([0.5, 0.9, 0.98, 1.0] if mesh.kind == "hex"
                             else [0.9, 1.0])
                elif A.nnz * 8 > 2**30:
                    fracs = [0.5, 1.0]
                else:
                    fracs = [1.0]
                fracs = fracs[-max(1, min(len(fracs), nl // 4)):]
                fracs[-1] = 1.0
                layers = slab_layers_fracs(mesh, fracs, None)
            plan = ColorPlan(mesh, None, self.device, work=work,
                             layers=layers)
        counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64,
                               device=self.device)
        if strategy == "blocked":
            self.build_blocks(A)
            if gather:
                self.block_a22(counters)
        d = space.degree
        plane = int(np.prod(space.grid_dims[:-1]))
        nplanes = int(space.grid_dims[-1])
        host = np.empty(A.nnz, dtype=np.float64)
        self._stream_host = host
        compute = torch.cuda.current_stream(self.device)
        ranges = []
        done_plane = 0
        for s_, (lo, hi) in enumerate(layers):
            if plan is not None:
                g0, g1 = plan.group_range(s_)
            final = nplanes if s_ == len(layers) - 1 else d * hi
            if gather:
                self.gather_blocks(A, done_plane * plane, final * plane)
            elif strategy == "blocked":
                self.scatter_blocks(A, plan, counters, groups=(g0, g1))
            else:
                self.run(A, plan=plan, counters=counters, flags=flags,
                         groups=(g0, g1))
            ev = torch.cuda.Event()
            ev.record(compute)
            a = int(A.rowptr[done_plane * plane])
            b = int(A.rowptr[final * plane])
            ranges.append((ev, a, b))
            done_plane = final
        src = A._dvals
        stager = HostStager(self.device)

        prefault = os.environ.get("MF_PREFAULT", "1") != "0"

        def worker():
            # first-touch the fresh result pages while the first range
            # computes, so the staged copies (and the exposed tail copy)
            # write into mapped memory.  Not on the gather path: its
            # kernels are as short as the prefault itself, so the copy
            # threads fault their own pages (measured the same 0.67 s on
            # R4 either way), and a prefault running beside the copies
            # would zero what they have already written.
            if prefault and not gather:
                stager.prefault(host)
            stager.run(src, host, ranges)

        self._stream_thread = threading.Thread(target=worker, daemon=True)
        self._stream_thread.start()
        return counters

    def join_streamed(self, A):
        self._stream_thread.join()
        A._vals = self._stream_host
        self._stream_host = None

    def build_blocks(self, A):
        """mf_offset_blocks: one Algorithm-1 run per (offset, proto pair) on
        the reference's synthetic geometry (_build_offset_blocks,
        _kernels.py:490-594); keeps the present blocks grouped by inner
        proto for the scatter."""
        import torch
        from . import _native as N
        from .device import to_device
        L = N.lib()
        mesh, space = self.mesh, self.space
        kind = mesh.kind
        kcode = {"quad": 0, "tri": 1, "hex": 2}[kind]
        nproto = 2 if kind == "tri" else 1
        nloc = 3 * space.degree if kind == "tri" else \
            (space.degree + 1) ** mesh.dim
        R = A._offset_reach
        dev = self.device
        nblk = int(L.mf_offset_block_count(mesh.dim, nproto, R))
        B21 = torch.empty(nblk * nloc * nloc, dtype=torch.float64, device=dev)
        B22 = torch.empty_like(B21)
        bev = torch.zeros(nblk, dtype=torch.int64, device=dev)
        protos = (to_device(_TRI_PROTOS, dev) if kind == "tri" else None)
        wsb = int(L.mf_offset_blocks_workspace_bytes(
            C_byref(self.drules.struct), nblk))
        ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
        N.check(L.mf_offset_blocks(
            C_byref(self.dmesh.struct), C_byref(self.drules.struct),
            C_byref(self.kernel_struct()), kcode, nproto, N.ptr(protos), R,
            float(mesh.h), N.ptr(B21), N.ptr(B22), N.ptr(bev), 0, N.ptr(ws),
            wsb, N.stream_ptr(device=self.device)), "mf_offset_blocks")
        ev = bev.cpu().numpy()
        ids = np.nonzero(ev > 0)[0]
        t1 = ids % nproto
        order = np.argsort(t1, kind="stable")
        blk = ids[order].astype(np.int32)
        blk_ptr = np.searchsorted(t1[order], np.arange(nproto + 1)).astype(
            np.int64)
        blk_d = to_device(blk if blk.size else np.zeros(1, np.int32), dev)
        self.n_blocks = int(blk.size)
        self._blocks = dict(B21=B21, B22=B22, bev=bev, blk=blk_d,
                            blk_ptr=blk_ptr, nproto=nproto, R=R)
        return self._blocks

    def scatter_blocks(self, A, plan, counters, scale=2.0, groups=None):
        """mf_scatter_offset_blocks over the colour groups of `plan`."""
        import torch
        from . import _native as N
        L = N.lib()
        b = self._blocks
        om = torch.ones(self.mesh.n_elements, dtype=torch.uint8,
                        device=self.device)
        g0, g1 = groups if groups is not None else (0, plan.ngroups)
        cptr = np.ascontiguousarray(plan.color_ptr[g0:g1 + 1])
        N.check(L.mf_scatter_offset_blocks(
            C_byref(self.dmesh.struct), C_byref(A._pattern_struct()),
            b["nproto"], b["R"], N.ptr(b["blk"]),
            b["blk_ptr"].ctypes.data_as(ctypes_void_p()), N.ptr(b["B21"]),
            N.ptr(b["B22"]), N.ptr(b["bev"]), N.ptr(om),
            N.ptr(plan.inner_sorted), cptr.ctypes.data_as(ctypes_void_p()),
            g1 - g0, float(scale), N.ptr(A._dvals), N.ptr(counters),
            N.stream_ptr(device=self.device)), "mf_scatter_offset_blocks")
        return counters

    def block_a22(self, counters):
        """Gather table + per-element sums of realised B22 blocks
        (mf_offset_block_a22)."""
        import torch
        from . import _native as N
        L = N.lib()
        b = self._blocks
        kcode = {"quad": 0, "tri": 1, "hex": 2}[self.mesh.kind]
        nloc = 3 if kcode == 1 else 2 ** self.mesh.dim
        b["a22"] = torch.empty(self.mesh.n_elements * nloc * nloc,
                               dtype=torch.float64, device=self.device)
        b["T"] = torch.empty(int(L.mf_gather_table_doubles(
            self.mesh.dim, kcode, b["R"])), dtype=torch.float64,
            device=self.device)
        b["kcode"] = kcode
        N.check(L.mf_offset_block_a22(
            C_byref(self.dmesh.struct), kcode, b["nproto"], b["R"],
            N.ptr(b["B21"]), N.ptr(b["B22"]), N.ptr(b["bev"]),
            N.ptr(b["a22"]), N.ptr(b["T"]), N.ptr(counters),
            N.stream_ptr(device=self.device)), "mf_offset_block_a22")

    def gather_blocks(self, A, row0, row1, scale=2.0):
        """Write vals rows [row0, row1) by the entry-wise gather
        (mf_gather_offset_blocks)."""
        from . import _native as N
        b = self._blocks
        N.check(N.lib().mf_gather_offset_blocks(
            C_byref(self.dmesh.struct), C_byref(A._pattern_struct()),
            b["kcode"], b["nproto"], b["R"], N.ptr(b["T"]), N.ptr(b["a22"]),
            int(row0), int(row1), float(scale), N.ptr(A._dvals),
            N.stream_ptr(device=self.device)), "mf_gather_offset_blocks")

    def run_blocked(self, A, scale=2.0, counters=None):
        """Offset-blocked strategy (assembly.py:391-437) on the device:
        the blocks, then the entry-wise gather (degree 1) or the
        colour-scheduled scatter (degree 2)."""
        import torch
        from . import _native as N
        from .device import ColorPlan
        self.build_blocks(A)
        if counters is None:
            counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64,
                                   device=self.device)
        if self.space.degree == 1:
            self.block_a22(counters)
            self.gather_blocks(A, 0, A.n, scale)
            return counters
        plan = ColorPlan(self.mesh, None, self.device)
        return self.scatter_blocks(A, plan, counters, scale)

    def finish(self, A, counters):
        """events/asymmetry/symmetrize (assembly.py:440-445, x2 folded)."""
        import torch
        from . import _native as N
        out = torch.zeros(1, dtype=torch.float64, device=self.device)
        pat = A._pattern_struct()
        N.check(N.lib().mf_asymmetry_inf(C_byref(pat), N.ptr(A._dvals),
                                          N.ptr(out), N.stream_ptr(device=self.device)),
                "mf_asymmetry_inf")
        if self.config.symmetrize:
            N.check(N.lib().mf_symmetrize(C_byref(pat), N.ptr(A._dvals),
                                           N.stream_ptr(device=self.device)), "mf_symmetrize")
        # wait on an event first: Event.synchronize releases the GIL, a
        # blocking .cpu() does not, and the streamed host copies
        # (run_streamed's worker threads) need it while the kernels run
        # (tools/overlap_probe.py: 8 GB staged in 3.23 s vs 0.23 s)
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream(self.device))
        done.synchronize()
        cnt = counters.cpu().numpy()
        check_counters(cnt)
        A.counters = cnt
        A.events = int(cnt[N.CNT_EVENTS])
        A.presym_asymmetry = float(out.item())
        return A


def check_counters(cnt):
    """Raise when a kernel flagged dropped work (MF_CNT_OVERFLOW): the
    values would be incomplete (include/mollifem_b200.h)."""
    from . import _native as N
    if int(cnt[N.CNT_OVERFLOW]):
        raise RuntimeError(
            "assembly kernel overflow: more split sub-cells per level than "
            "the specialised kernel buffers; the matrix is incomplete "
            "(use flags=MF_FLAG_FORCE_GENERIC)")


class WindowedValues:
    """A device tensor holding vals[base : base + n] of a larger pattern.

    The kernels index vals with absolute pattern offsets, so they get the
    tensor's address shifted back by `base` elements; every offset they
    touch (rows of the caller's inner elements) lies inside the window."""

    def __init__(self, tensor, base):
        self.tensor = tensor
        self.base = int(base)

    def pointer(self):
        import ctypes
        return ctypes.c_void_p(self.tensor.data_ptr() - 8 * self.base)


def ctypes_void_p():
    import ctypes
    return ctypes.c_void_p


# lower (sw, se, ne) and upper (sw, ne, nw) triangle protos in cell units
# (assembly.py:44-48)
_TRI_PROTOS = np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]],
                        [[0.0, 0.0], [1.0, 1.0], [0.0, 1.0]]])


def resolve_strategy(mesh, config):
    """assembly.py:448-453: "auto" -> blocked on pure quad/tri/hex meshes.

    Tet and Delaunay meshes (new) always run the general path: their
    elements have no translation-invariant offset blocks."""
    unstructured = getattr(mesh, "unstructured", False)
    if config.strategy == "blocked" and (
            unstructured or mesh.kind not in ("quad", "tri", "hex")):
        raise ValueError("blocked strategy needs a pure structured "
                         "quad/tri/hex mesh")
    if config.strategy != "auto":
        return config.strategy
    if unstructured:
        return "general"
    return "blocked" if mesh.kind in ("quad", "tri", "hex") else "general"


def assemble(mesh, space, kernel, config=None, *, device=None, flags=0,
             keep_on_device=False):
    """Assemble the stiffness matrix A = 2(A21 + A22) on the GPU.

    Same arguments and return contract as the reference (assembly.py:456):
    a `SparseMatrix` with host `vals` (already x2), `events` and
    `presym_asymmetry`.  Strategy resolution follows the reference: "auto"
    runs the offset-blocked path on pure quad/tri/hex meshes, "general" the
    per-pair path (mf_general_core).  keep_on_device=True skips the host copy (the
    values stay in `A.vals_device`; `A.vals` copies them on first use).
    """
    import torch
    from .device import _dev
    config = config or AssemblyConfig()
    if config.method == "barycenter":
        raise NotImplementedError(
            "the barycenter baseline (assembly.py:565-635) is outside the "
            "B200 hot path; use the reference package for it")
    dev = _dev(device)
    with torch.cuda.device(dev):
        return _assemble_on(mesh, space, kernel, config, dev, flags,
                            keep_on_device)


def _assemble_on(mesh, space, kernel, config, device, flags, keep_on_device):
    ctx = AssemblyContext(mesh, space, kernel, config, device)
    A = ctx.new_matrix()
    strategy = resolve_strategy(mesh, config)
    if keep_on_device or config.symmetrize or A.nnz * 8 < _STREAM_MIN_BYTES:
        counters = (ctx.run_blocked(A) if strategy == "blocked"
                    else ctx.run(A, flags=flags))
        ctx.finish(A, counters)
        if not keep_on_device:
            A._vals = _d2h(A._dvals)
        return A
    counters = ctx.run_streamed(A, flags=flags, strategy=strategy)
    ctx.finish(A, counters)
    ctx.join_streamed(A)
    return A


# ---------------------------------------------------------------------------
# load vector (assembly.py:641-691)

def _load_points(mesh, space, sel, code):
    """Physical rule points of elements `sel` of kind `code` and the rule
    (GL(degree+2) on boxes, Dunavant on triangles; assembly.py:648-669)."""
    from .fe_space import eval_shape_functions
    deg = space.degree
    box_kind = "hex" if mesh.dim == 3 else "quad"
    if code == 3:
        # tetrahedra (new element): degree-4 Keast rule, affine map
        rule = rule_for_kind("tet", "tet11")
        kname = "tet"
        v = mesh.elem_coords[sel, :4, :]
        E = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0],
                      v[:, 3] - v[:, 0]], axis=2)
        pts = v[:, None, 0, :] + np.einsum("ekj,qj->eqk", E, rule.ref_points)
    elif code == 1:
        rule = rule_for_kind("tri", "default")
        kname = "tri"
        v = mesh.elem_coords[sel, :3, :]
        e1 = v[:, 1] - v[:, 0]
        e2 = v[:, 2] - v[:, 0]
        r = rule.ref_points
        pts = (v[:, None, 0, :] + r[None, :, 0, None] * e1[:, None, :]
               + r[None, :, 1, None] * e2[:, None, :])
    else:
        rule = rule_for_kind(box_kind, "gauss" + str(deg + 2))
        kname = box_kind
        lo = mesh.elem_lo[sel]
        hi = mesh.elem_hi[sel]
        r = rule.ref_points
        pts = lo[:, None, :] + (r[None, :, :] + 1.0) * 0.5 * (hi - lo)[:, None, :]
    PHI = eval_shape_functions(kname, deg, rule.ref_points)
    return pts, rule, PHI


def group_load_device(mesh, space, f, element_ids, dmesh, device=None):
    """(int_Omega f phi) for `element_ids` as a device vector
    (_group_load, assembly.py:641-676): f is evaluated on the host at the
    rule points, the contraction and the colour-scheduled scatter run in
    mf_load_scatter."""
    import torch
    from . import _native as N
    from .device import color_of, ncolors_of, to_device
    L = N.lib()
    dev = dmesh.device
    load = torch.zeros(space.n_dofs, dtype=torch.float64, device=dev)
    kinds = mesh.elem_kind
    col = color_of(mesh)
    for code in (0, 1, 2, 3):
        sel = element_ids[kinds[element_ids] == code]
        if len(sel) == 0:
            continue
        sel = sel[np.argsort(col[sel], kind="stable")]
        pts, rule, PHI = _load_points(mesh, space, sel, code)
        fv = np.asarray(f(pts.reshape(-1, mesh.dim)), dtype=float)
        fv = np.ascontiguousarray(np.broadcast_to(
            fv, (pts.shape[0] * pts.shape[1],)).reshape(len(sel), len(rule)))
        ncol = ncolors_of(mesh)
        counts = np.bincount(col[sel], minlength=ncol)
        cptr = np.zeros(ncol + 1, dtype=np.int64)
        np.cumsum(counts, out=cptr[1:])
        elems = to_device(sel.astype(np.int32), dev)
        fvd = to_device(fv, dev)
        wd = to_device(np.ascontiguousarray(rule.weights), dev)
        phid = to_device(np.ascontiguousarray(PHI), dev)
        N.check(L.mf_load_scatter(
            C_byref(dmesh.struct), N.ptr(elems),
            cptr.ctypes.data_as(ctypes_void_p()), ncol,
            N.ptr(fvd), N.ptr(wd), N.ptr(phid), len(rule), PHI.shape[1],
            N.ptr(load), N.stream_ptr(device=dev)), "mf_load_scatter")
    return load


def assemble_rhs(mesh, space, kernel, f, g, A):
    """rhs = (int_Omega f phi)[free] - (A gt)[free] (assembly.py:679-691).

    gt is the nodal interpolant of g on constrained DOFs (callable, or an
    array over all DOFs / constrained DOFs), zero elsewhere."""
    import torch
    dev = A.vals_device.device
    with torch.cuda.device(dev):
        return _assemble_rhs_on(mesh, space, f, g, A, dev)


def _assemble_rhs_on(mesh, space, f, g, A, dev):
    import torch
    from . import _native as N
    from .device import DeviceMesh, to_device
    dmesh = DeviceMesh(mesh, space, dev)
    load = group_load_device(mesh, space, f, mesh.omega_element_ids(), dmesh)
    gt = np.zeros(space.n_dofs)
    if callable(g):
        gt[space.constrained] = g(space.dof_coords[space.constrained])
    else:
        gv = np.asarray(g, dtype=float)
        gt[space.constrained] = (gv[space.constrained]
                                 if gv.shape == (space.n_dofs,) else gv)
    gtd = to_device(gt, dev)
    y = torch.empty_like(gtd)
    st = N.stream_ptr(device=dev)
    L = N.lib()
    N.check(L.mf_matvec(C_byref(A._pattern_struct()), N.ptr(A.vals_device),
                        N.ptr(gtd), N.ptr(y), st), "mf_matvec")
    free = np.asarray(space.free, dtype=np.int64)
    free_d = to_device(free, dev)
    out = torch.empty(len(free), dtype=torch.float64, device=dev)
    N.check(L.mf_gather_diff(len(free), N.ptr(free_d), N.ptr(load), N.ptr(y),
                             N.ptr(out), st), "mf_gather_diff")
    return out.cpu().numpy()
