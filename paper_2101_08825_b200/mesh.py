"""Structured meshes of Omega plus its constraint layer (reference row a3).

Restates `mollifem/mesh.py:75-319` with vectorised construction: the same
flat SoA arrays (`elem_kind`, `elem_proto`, `elem_region`, `elem_cell`,
`elem_coords`, `elem_lo`, `elem_hi`), bit-identical coordinates
(`origin + h*arange`, mesh.py:180-191), the same cell-lex element order
(tri cells emit the lower then the upper triangle) and the same recursive
coordinate bisection.  `Mesh.elements` is materialised lazily, so building
the 474,552-hex R4 mesh takes well under a second instead of the
reference's per-element Python loop.
"""

import math

import numpy as np

__all__ = ["BoundingBox", "DelaunayMesh", "Element", "Mesh", "PartitionMap",
           "build_delaunay_mesh", "build_mesh", "refine",
           "partition_geometric"]

KIND_CODE = {"quad": 0, "tri": 1, "hex": 2, "tet": 3}
KIND_NAME = {0: "quad", 1: "tri", 2: "hex", 3: "tet"}

# 6-tet (Kuhn / Freudenthal) split of a cube: tet p follows the axis
# permutation KUHN_PERMS[p] from corner 0 to corner 7 (corner bit k = axis
# k).  The triangulation is conforming across cubes.  Odd permutations swap
# their middle vertices so that every tet is positively oriented.
KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1),
              (2, 1, 0))


def kuhn_corners(p):
    """Cube corner ids (bit k = axis k) of Kuhn tet p, positive orientation."""
    a, b, _ = KUHN_PERMS[p]
    v1 = 1 << a
    v2 = v1 | (1 << b)
    odd = p in (1, 2, 5)
    return (0, v2, v1, 7) if odd else (0, v1, v2, 7)


class BoundingBox:
    """Axis-aligned box (lo, hi)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        self.lo = np.asarray(lo, dtype=float)
        self.hi = np.asarray(hi, dtype=float)
        if np.any(self.lo > self.hi):
            raise ValueError("box needs lo <= hi componentwise")

    @property
    def center(self):
        return 0.5 * (self.lo + self.hi)

    def contains(self, point, tol=0.0):
        p = np.asarray(point, dtype=float)
        return bool(np.all(p >= self.lo - tol) and np.all(p <= self.hi + tol))

    def __repr__(self):
        return f"BoundingBox({self.lo.tolist()}, {self.hi.tolist()})"


class Element:
    """One element: geometry node ids/coords, region tag and bbox."""

    __slots__ = ("id", "kind", "node_ids", "region", "bbox", "coords")

    def __init__(self, eid, kind, node_ids, region, coords):
        self.id = eid
        self.kind = kind
        self.node_ids = node_ids
        self.region = region
        self.coords = coords
        self.bbox = BoundingBox(coords.min(axis=0), coords.max(axis=0))

    def measure(self):
        if self.kind == "tri":
            a = self.coords[1] - self.coords[0]
            b = self.coords[2] - self.coords[0]
            return 0.5 * abs(a[0] * b[1] - a[1] * b[0])
        if self.kind == "tet":
            e = self.coords[1:4] - self.coords[0]
            return abs(float(np.linalg.det(e))) / 6.0
        return float(np.prod(self.bbox.hi - self.bbox.lo))

    def __repr__(self):
        return f"Element({self.id}, {self.kind}, {self.region})"


class _LazyElements:
    """Sequence view that builds `Element` records on demand."""

    def __init__(self, mesh):
        self._m = mesh

    def __len__(self):
        return self._m.elem_kind.shape[0]

    def __getitem__(self, i):
        m = self._m
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        k = int(m.elem_kind[i])
        nv = 3 if k == 1 else m.elem_nodes.shape[1]
        ids = m.elem_nodes[i, :nv].copy()
        return Element(i, KIND_NAME[k], ids,
                       "omega" if m.elem_region[i] == 0 else "gamma",
                       m.nodes[ids])

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class Mesh:
    """Structured mesh; see module docstring for the flat arrays."""

    def __init__(self, dim, nodes, elem_nodes, h, omega_bounds, gamma_layers,
                 kind, layer_width, grid_ncells, grid_origin, arrays,
                 jitter=0.0, seed=0):
        self.dim = dim
        self.jitter = float(jitter)      # fraction of h (tet meshes only)
        self.seed = int(seed)
        self.nodes = nodes
        self.elem_nodes = elem_nodes
        self.h = h
        self.omega_bounds = omega_bounds
        self.gamma_layers = gamma_layers
        self.kind = kind
        self.layer_width = layer_width
        self.grid_ncells = grid_ncells
        self.grid_origin = grid_origin
        (self.elem_kind, self.elem_proto, self.elem_region, self.elem_cell,
         self.elem_coords, self.elem_lo, self.elem_hi) = arrays
        self.elements = _LazyElements(self)

    @property
    def n_elements(self):
        return int(self.elem_kind.shape[0])

    @property
    def stencil_pad(self):
        """Extra reach of the cell stencil: element boxes of a jittered mesh
        stick out of their cells by up to jitter*h on every side."""
        return 2.0 * self.jitter * self.h

    def omega_element_ids(self):
        return np.nonzero(self.elem_region == 0)[0]

    def domain_bounds(self):
        lo = np.asarray(self.grid_origin)
        return BoundingBox(lo, lo + np.asarray(self.grid_ncells) * self.h)

    def cell_flat(self):
        """Flat cell id per element, x fastest (assembly.py:135-141)."""
        c = self.elem_cell.astype(np.int64)
        nc = self.grid_ncells
        flat = c[:, 1] * nc[0] + c[:, 0]
        if self.dim == 3:
            flat += c[:, 2] * (nc[0] * nc[1])
        return flat.astype(np.int32)

    def cell_ptr(self):
        """CSR of elements per flat cell (elements are cell-lex ordered)."""
        flat = self.cell_flat()
        ncells = int(np.prod(self.grid_ncells))
        return flat, np.searchsorted(flat, np.arange(ncells + 1)).astype(
            np.int64)

    def __repr__(self):
        return (f"Mesh(dim={self.dim}, kind={self.kind}, h={self.h}, "
                f"elements={self.n_elements}, rings={self.gamma_layers})")


class PartitionMap:
    """Element -> part map with per-part bounding boxes."""

    def __init__(self, n_parts, owner, part_bbox):
        self.n_parts = n_parts
        self.owner = owner
        self.part_bbox = part_bbox

    def owned(self, part):
        return np.nonzero(self.owner == part)[0]

    def __repr__(self):
        return f"PartitionMap(n_parts={self.n_parts})"


def _as_bounds(omega_bounds, dim):
    if isinstance(omega_bounds, BoundingBox):
        lo, hi = omega_bounds.lo, omega_bounds.hi
    else:
        arr = np.asarray(omega_bounds, dtype=float)
        if arr.shape != (dim, 2):
            raise ValueError(f"omega_bounds must be {dim} (lo, hi) pairs")
        lo, hi = arr[:, 0], arr[:, 1]
    if len(lo) != dim:
        raise ValueError("omega_bounds dimension mismatch")
    return BoundingBox(lo, hi)


def build_mesh(dim, omega_bounds, h, layer_width, kind="quad", jitter=0.0,
               seed=0):
    """Omega tiled at pitch h plus ceil(layer_width/h) Gamma rings.

    kind: quad/tri/mixed in 2D (mesh.py:153-165); hex or tet in 3D.  "tet"
    (new, BASELINE configs #4/#5; the reference has no tetrahedra) splits
    every cube into the 6 Kuhn tets.  jitter (tet only) moves every vertex
    coordinate by a seeded uniform offset in [-jitter*h, jitter*h], except
    along axes where the vertex lies on the outer boundary or on an
    Omega/Gamma interface plane, so the regions stay exact boxes.
    """
    if h <= 0.0:
        raise ValueError("h must be positive")
    if layer_width < 0.0:
        raise ValueError("layer_width must be nonnegative")
    rings = int(math.ceil(layer_width / h - 1e-9)) if layer_width > 0.0 else 0
    return _build(dim, omega_bounds, h, rings, kind, layer_width, jitter,
                  seed)


def _build(dim, omega_bounds, h, rings, kind, layer_width, jitter=0.0,
           seed=0):
    if dim == 2 and kind not in ("quad", "tri", "mixed"):
        raise ValueError(f"2D mesh kind must be quad/tri/mixed, got {kind!r}")
    if dim == 3 and kind not in ("hex", "tet"):
        raise ValueError("3D meshes are hex or tet")
    if jitter and kind != "tet":
        raise ValueError("jitter is supported for tet meshes only")
    if not 0.0 <= jitter <= 0.2:
        raise ValueError("jitter must lie in [0, 0.2] (tets stay valid)")
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    box = _as_bounds(omega_bounds, dim)
    side = box.hi - box.lo
    n_omega = np.rint(side / h).astype(int)
    if np.any(n_omega < 1) or np.any(
            np.abs(n_omega * h - side) > 1e-9 * np.maximum(1.0, side)):
        raise ValueError(f"omega side lengths {side.tolist()} are not "
                         f"integer multiples of h={h}")
    nc = n_omega + 2 * rings
    origin = box.lo - rings * h
    nv = nc + 1
    axes = [origin[k] + h * np.arange(nv[k]) for k in range(dim)]
    grids = np.meshgrid(*axes[::-1], indexing="ij")      # z/y slowest
    nodes = np.column_stack([g.ravel() for g in grids[::-1]])

    # per-cell integer coordinates, x fastest
    cidx = np.indices(tuple(nc[::-1])).reshape(dim, -1)[::-1].T  # (ncell,dim)
    inside = np.all((cidx >= rings) & (cidx < rings + n_omega), axis=1)
    region_c = np.where(inside, 0, 1).astype(np.int8)

    def nid(off):
        g = cidx + np.asarray(off)[None, :]
        out = g[:, -1].astype(np.int64)
        for k in range(dim - 2, -1, -1):
            out = out * nv[k] + g[:, k]
        return out

    if dim == 3 and kind == "tet":
        corners = [((v & 1), (v >> 1) & 1, (v >> 2) & 1) for v in range(8)]
        cn = np.stack([nid(c) for c in corners], axis=1)      # (ncell, 8)
        # 6 tets per cube, cube-major (cell-lex order of the elements)
        tets = np.array([kuhn_corners(p) for p in range(6)])  # (6, 4)
        en = cn[:, tets].reshape(-1, 4)
        kinds = np.full(en.shape[0], 3, np.int8)
        protos = np.tile(np.arange(6, dtype=np.int8), len(cidx))
        cells = np.repeat(cidx, 6, axis=0)
        regions = np.repeat(region_c, 6)
        if jitter > 0.0:
            rng = np.random.default_rng(seed)
            gidx = np.indices(tuple(nv[::-1])).reshape(dim, -1)[::-1].T
            off = rng.uniform(-jitter * h, jitter * h, size=nodes.shape)
            fixed = ((gidx == 0) | (gidx == nv[None, :] - 1)
                     | (gidx == rings) | (gidx == rings + n_omega[None, :]))
            nodes = nodes + np.where(fixed, 0.0, off)
    elif dim == 3:
        corners = [((v & 1), (v >> 1) & 1, (v >> 2) & 1) for v in range(8)]
        en = np.stack([nid(c) for c in corners], axis=1)
        kinds = np.full(len(cidx), 2, np.int8)
        protos = np.zeros(len(cidx), np.int8)
        cells = cidx
        regions = region_c
    else:
        sw, se, nw, ne = (nid((0, 0)), nid((1, 0)), nid((0, 1)),
                          nid((1, 1)))
        if kind == "quad":
            as_quad = np.ones(len(cidx), bool)
        elif kind == "tri":
            as_quad = np.zeros(len(cidx), bool)
        else:
            as_quad = (cidx[:, 0] + cidx[:, 1]) % 2 == 0
        nvmax = 4 if as_quad.any() else 3
        # two slots per cell: slot 0 = quad or lower tri, slot 1 = upper tri
        slot_nodes = np.zeros((len(cidx), 2, nvmax), np.int64)
        q = as_quad
        t = ~as_quad
        if q.any():
            slot_nodes[q, 0, :4] = np.stack([sw, se, nw, ne], 1)[q]
        slot_nodes[t, 0, :3] = np.stack([sw, se, ne], 1)[t]
        slot_nodes[t, 1, :3] = np.stack([sw, ne, nw], 1)[t]
        valid = np.stack([np.ones(len(cidx), bool), t], axis=1)
        sel = valid.ravel()
        en = slot_nodes.reshape(-1, nvmax)[sel]
        kinds = np.stack([np.where(q, 0, 1), np.ones(len(cidx), int)],
                         1).ravel()[sel].astype(np.int8)
        protos = np.stack([np.zeros(len(cidx), int), np.ones(len(cidx), int)],
                          1).ravel()[sel].astype(np.int8)
        cells = np.repeat(cidx, 2, axis=0)[sel]
        regions = np.repeat(region_c, 2)[sel]

    n_elem = en.shape[0]
    nvmax = en.shape[1]
    coords = nodes[en]                                   # (n, nvmax, dim)
    is_tri = kinds == 1
    if is_tri.any() and nvmax > 3:
        coords[is_tri, 3:, :] = 0.0
    lo = np.where(is_tri[:, None], coords[:, :3, :].min(axis=1),
                  coords.min(axis=1))
    hi = np.where(is_tri[:, None], coords[:, :3, :].max(axis=1),
                  coords.max(axis=1))
    arrays = (kinds, protos, regions.astype(np.int8),
              cells.astype(np.int32), np.ascontiguousarray(coords),
              np.ascontiguousarray(lo), np.ascontiguousarray(hi))
    return Mesh(dim, nodes, en, h, box, rings, kind, layer_width,
                tuple(int(x) for x in nc), origin, arrays, jitter, seed)


def refine(mesh):
    """Uniform refinement: h halves, ring count doubles."""
    return _build(mesh.dim, mesh.omega_bounds, mesh.h / 2.0,
                  mesh.gamma_layers * 2, mesh.kind, mesh.layer_width,
                  mesh.jitter, mesh.seed)


def partition_geometric(mesh, n_parts):
    """Recursive coordinate bisection of element centroids (mesh.py:284-319).

    Widest centroid axis, stable median split, proportional counts.
    """
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    n_elem = mesh.n_elements
    if n_parts > n_elem:
        raise ValueError("n_parts exceeds element count")
    cen = 0.5 * (mesh.elem_lo + mesh.elem_hi)
    owner = np.empty(n_elem, dtype=np.int32)
    stack = [(np.arange(n_elem), n_parts, 0)]
    while stack:
        ids, parts, first = stack.pop()
        if parts == 1:
            owner[ids] = first
            continue
        n1 = (parts + 1) // 2
        count1 = (len(ids) * n1) // parts
        sub = cen[ids]
        axis = int(np.argmax(sub.max(axis=0) - sub.min(axis=0)))
        order = np.argsort(sub[:, axis], kind="stable")
        stack.append((ids[order[count1:]], parts - n1, first + n1))
        stack.append((ids[order[:count1]], n1, first))
    boxes = []
    for p in range(n_parts):
        ids = np.nonzero(owner == p)[0]
        boxes.append(BoundingBox(mesh.elem_lo[ids].min(axis=0),
                                 mesh.elem_hi[ids].max(axis=0)))
    return PartitionMap(n_parts, owner, boxes)


# ---------------------------------------------------------------------------
# unstructured Delaunay triangle meshes (BASELINE config #2; new -- the
# reference builds structured meshes only, mesh.py:153-178)

class DelaunayMesh(Mesh):
    """Delaunay P1 triangulation of jittered lattice points.

    Every vertex is drawn from one lattice node of pitch h (uniform offset
    in [-jitter*h, jitter*h] per axis) and keeps that node's lattice index
    as its id, so the DOF numbering and the implicit box pattern of the
    structured path apply unchanged.  The triangulation itself is
    unstructured: connectivity, valence and element shapes come from
    scipy's Delaunay (qhull).  Elements are binned by the lattice cell of
    their bounding-box lower corner and stored in bin-lex order, which is
    the cell ordering the neighbour search and the kernels walk.

    Extra attributes over `Mesh`:
      unstructured  True
      emax          largest element box side (<= 2h is asserted)
      elem_color    greedy colouring: elements of one colour share no vertex
      n_colors      number of colours
      row_period    stencil rows this far apart hold outer elements that
                    share no vertex (3, since emax <= 2h)
    """

    unstructured = True
    row_period = 3

    @property
    def stencil_pad(self):
        # element boxes reach emax beyond the lower corner that bins them
        return self.emax

    @property
    def pattern_pad(self):
        # coupled vertices lie within reach + 2 emax of each other, and a
        # vertex within jitter*h of its lattice node
        return 2.0 * self.emax + 2.0 * self.jitter * self.h


def _greedy_colors(elem_nodes, n_nodes, seed=0):
    """Jones-Plassmann colouring of the element/vertex-sharing graph:
    each round, every uncoloured element whose random priority beats all
    its uncoloured neighbours takes the smallest colour no neighbour has.
    Deterministic for a seed; about max-degree+1 colours at most."""
    n, nv = elem_nodes.shape
    flat = elem_nodes.ravel()
    eid = np.repeat(np.arange(n), nv)
    order = np.argsort(flat, kind="stable")
    vptr = np.searchsorted(flat[order], np.arange(n_nodes + 1))
    ve = eid[order]
    # element pairs sharing a vertex
    cnt = np.diff(vptr)
    src, dst = [], []
    for k in range(1, int(cnt.max()) if cnt.size else 1):
        has = np.nonzero(cnt > k)[0]
        for j in range(k):
            a = ve[vptr[has] + k]
            b = ve[vptr[has] + j]
            src += [a, b]
            dst += [b, a]
    src = np.concatenate(src) if src else np.zeros(0, np.int64)
    dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
    # (pairs sharing two vertices appear twice; harmless below)
    src0, dst0 = src, dst
    rng = np.random.default_rng(seed)
    prio = rng.permutation(n)
    color = np.full(n, -1, dtype=np.int64)
    while True:
        unc = color < 0
        if not unc.any():
            break
        # keep only edges out of uncoloured elements
        keep = unc[src]
        src, dst = src[keep], dst[keep]
        # an uncoloured neighbour with higher priority -> wait this round
        blocked = np.zeros(n, dtype=bool)
        sel = unc[dst] & (prio[dst] > prio[src])
        blocked[src[sel]] = True
        pick = unc & ~blocked
        # colours used by coloured neighbours (bit mask, < 63 colours)
        used = np.zeros(n, dtype=np.int64)
        cs = ~unc[dst] & pick[src]
        np.bitwise_or.at(used, src[cs], np.int64(1) << color[dst[cs]])
        ids = np.nonzero(pick)[0]
        u = used[ids]
        if (u >= np.int64(1) << 61).any() or (u < 0).any():
            # int64 masks hold 61 colours safely (1 << 62 would overflow)
            raise RuntimeError("greedy colouring needs more than 61 colours")
        low = ~u & (u + 1)               # lowest clear bit = smallest free
        color[ids] = np.log2(low.astype(np.float64)).astype(np.int64)
    # every colour class must be vertex-disjoint (the kernels' writes to a
    # colour are non-atomic): no edge may join two elements of one colour
    if (color[src0] == color[dst0]).any():
        raise RuntimeError("colouring is not vertex-disjoint")
    return color


def build_delaunay_mesh(omega_bounds, h, layer_width, jitter=0.3, seed=0):
    """Unstructured Delaunay P1 mesh of Omega plus ceil(layer_width/h)
    Gamma rings (BASELINE config #2: seeded uniform jittered vertices).

    Lattice nodes of pitch h are moved by a seeded uniform offset in
    [-jitter*h, jitter*h] per axis; nodes on the outer boundary or on the
    Omega/Gamma interface keep that coordinate and move along their line
    by at most jitter*h/2.  Each interface segment is then a Gabriel edge
    (its diametral circle, radius <= (1+jitter)h/2, holds no other node),
    so it is a Delaunay edge and every triangle lies in Omega or in Gamma;
    the builder checks this, the orientation and emax <= 2h.
    """
    from scipy.spatial import Delaunay
    if not 0.0 <= jitter <= 0.35:
        raise ValueError("jitter must lie in [0, 0.35]")
    if h <= 0.0 or layer_width < 0.0:
        raise ValueError("need h > 0 and layer_width >= 0")
    dim = 2
    box = _as_bounds(omega_bounds, dim)
    side = box.hi - box.lo
    n_omega = np.rint(side / h).astype(int)
    if np.any(n_omega < 1) or np.any(
            np.abs(n_omega * h - side) > 1e-9 * np.maximum(1.0, side)):
        raise ValueError(f"omega side lengths {side.tolist()} are not "
                         f"integer multiples of h={h}")
    rings = int(math.ceil(layer_width / h - 1e-9)) if layer_width > 0.0 else 0
    nc = n_omega + 2 * rings
    nv = nc + 1
    origin = box.lo - rings * h
    gy, gx = np.meshgrid(np.arange(nv[1]), np.arange(nv[0]), indexing="ij")
    gidx = np.stack([gx.ravel(), gy.ravel()], axis=1)     # lattice-lex ids
    base = origin[None, :] + h * gidx
    rng = np.random.default_rng(seed)
    off = rng.uniform(-jitter * h, jitter * h, size=base.shape)
    fixed = ((gidx == 0) | (gidx == nv[None, :] - 1) | (gidx == rings)
             | (gidx == rings + n_omega[None, :]))
    online = fixed.any(axis=1, keepdims=True)
    off = np.where(fixed, 0.0, np.where(online, 0.5 * off, off))
    nodes = base + off
    tri = Delaunay(nodes)
    en = np.ascontiguousarray(tri.simplices.astype(np.int64))
    c = nodes[en]
    det = ((c[:, 1, 0] - c[:, 0, 0]) * (c[:, 2, 1] - c[:, 0, 1])
           - (c[:, 1, 1] - c[:, 0, 1]) * (c[:, 2, 0] - c[:, 0, 0]))
    flip = det < 0.0
    en[flip] = en[flip][:, [0, 2, 1]]                    # counter-clockwise
    # canonical vertex order: smallest id first (rotation keeps the
    # orientation), so the element arrays depend only on the triangulation
    first = np.argmin(en, axis=1)
    rot = (first[:, None] + np.arange(3)[None, :]) % 3
    en = np.take_along_axis(en, rot, axis=1)
    if np.any(np.abs(det) < 1e-6 * h * h):
        raise RuntimeError("degenerate Delaunay triangle")
    c = nodes[en]
    lo = c.min(axis=1)
    hi = c.max(axis=1)
    emax = float((hi - lo).max())
    if emax > 2.0 * h:
        raise RuntimeError(f"element extent {emax / h:.3f} h exceeds 2h")
    cen = c.mean(axis=1)
    in_omega = np.all((cen > box.lo) & (cen < box.hi), axis=1)
    vin = np.all((c >= box.lo - 1e-12) & (c <= box.hi + 1e-12), axis=(1, 2))
    vstrict = np.all((c > box.lo) & (c < box.hi), axis=2).any(axis=1)
    if np.any(in_omega & ~vin) or np.any(~in_omega & vstrict):
        raise RuntimeError("a triangle straddles the Omega/Gamma interface")
    # bin by the lattice cell of the box lower corner; bin-lex order
    cell = np.floor((lo - origin[None, :]) / h).astype(np.int64)
    cell = np.clip(cell, 0, nc[None, :] - 1)
    order = np.lexsort((en[:, 2], en[:, 1], en[:, 0], cell[:, 0],
                        cell[:, 1]))
    en, c, lo, hi, cell = en[order], c[order], lo[order], hi[order], \
        cell[order]
    in_omega = in_omega[order]
    n = en.shape[0]
    arrays = (np.full(n, 1, np.int8), np.zeros(n, np.int8),
              np.where(in_omega, 0, 1).astype(np.int8),
              cell.astype(np.int32), np.ascontiguousarray(c),
              np.ascontiguousarray(lo), np.ascontiguousarray(hi))
    m = DelaunayMesh(dim, nodes, en, h, box, rings, "tri", layer_width,
                     tuple(int(x) for x in nc), origin, arrays, jitter, seed)
    m.emax = emax
    # lattice planes a vertex sits above its element's bin row (top axis)
    m.dof_spill = int((en // nv[0] - cell[:, 1:2]).max())
    if (en // nv[0] - cell[:, 1:2]).min() < 0:
        raise RuntimeError("a vertex lies below its element's bin row")
    m.elem_color = _greedy_colors(en, nodes.shape[0], seed)
    m.n_colors = int(m.elem_color.max()) + 1
    return m
