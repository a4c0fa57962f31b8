"""Triangle meshes, connectivity and per-element affine geometry.

Host-side setup for the stage kernels.  The public surface mirrors the
reference ``qfswe.mesh`` (mesh.py:19-31): ``Mesh``, ``Edge``,
``build_square_mesh``, ``build_ring_mesh``, ``compute_geometry``,
``load_mesh``/``save_mesh`` and the same exception types, with the same
conventions:

* triangles are counter-clockwise; local edge j is opposite local vertex j,
  i.e. (a1,a2), (a2,a0), (a0,a1) (mesh.py:84);
* ``mesh.edges`` is in first-encounter order of the (triangle, local edge)
  loop; the first triangle is the edge's *left* side, the second its
  *right* side, which must traverse the edge in the opposite direction
  (mesh.py:79-107);
* edge normal = outward normal of the left triangle, (dy, -dx)/len of
  v1 - v0 (mesh.py:272-278); B = [a2-a1, a3-a1] (mesh.py:262-264).

Unlike the reference (a Python dict loop over edges, mesh.py:83-102), the
connectivity is built with sorted integer keys in numpy so that 33.5M-element
meshes set up in seconds, and it is stored as flat arrays; ``mesh.edges``
materialises ``Edge`` objects lazily for small-mesh compatibility.

Added generators for the BASELINE configurations: ``build_unit_square_mesh``
(unit square, every quad split SW-NE, optional interior-only SplitMix64
jitter) — SURVEY §8d C1-C5.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

__all__ = [
    "DegenerateElement",
    "MeshParseError",
    "ConnectivityError",
    "Edge",
    "Mesh",
    "ElementGeometry",
    "EdgeGeometry",
    "build_square_mesh",
    "build_unit_square_mesh",
    "build_ring_mesh",
    "compute_geometry",
    "load_mesh",
    "save_mesh",
    "DIRICHLET",
    "locality_order",
]

DIRICHLET = 1
FORMAT_HEADER = "ghoddess-mesh 1"
_LOCAL = ((1, 2), (2, 0), (0, 1))  # local edge j = (a_{j+1}, a_{j+2})


class DegenerateElement(ValueError):
    """Triangle with non-positive Jacobian determinant."""


class MeshParseError(ValueError):
    """Malformed mesh file; message carries the line number."""


class ConnectivityError(ValueError):
    """Non-manifold or inconsistent triangle connectivity."""


@dataclass
class Edge:
    v0: int
    v1: int
    left: int
    left_local: int
    right: int = -1
    right_local: int = -1
    marker: int = 0

    @property
    def is_boundary(self) -> bool:
        return self.right < 0


@dataclass
class Connectivity:
    """Flat edge and element-neighbour tables (all int64)."""

    v0: np.ndarray
    v1: np.ndarray
    left: np.ndarray
    left_local: np.ndarray
    right: np.ndarray
    right_local: np.ndarray
    marker: np.ndarray        # 0 for interior edges
    elem_edge: np.ndarray     # (E, 3) edge index of each local edge
    nbr: np.ndarray           # (E, 3) neighbour element, -1 on the boundary
    nbr_local: np.ndarray     # (E, 3) neighbour's local edge, or -marker

    @property
    def n_edges(self) -> int:
        return len(self.v0)


@dataclass
class Mesh:
    vertices: np.ndarray      # (NV, 2) float64
    triangles: np.ndarray     # (E, 3) int64, counter-clockwise
    boundary_markers: dict = field(default_factory=dict)
    _conn: Connectivity | None = field(default=None, repr=False)
    _edges_cache: list | None = field(default=None, repr=False)

    @property
    def conn(self) -> Connectivity:
        """Flat connectivity tables (built on first use for lazily built meshes)."""
        if self._conn is None:
            build_connectivity(self)
        return self._conn

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)

    @property
    def edges(self) -> list[Edge]:
        """Reference-compatible list of ``Edge`` objects (built lazily)."""
        if self._edges_cache is None:
            c = self.conn
            self._edges_cache = [
                Edge(int(c.v0[i]), int(c.v1[i]), int(c.left[i]), int(c.left_local[i]),
                     int(c.right[i]), int(c.right_local[i]), int(c.marker[i]))
                for i in range(c.n_edges)
            ]
        return self._edges_cache


def build_connectivity(mesh: Mesh) -> None:
    """Vectorised equivalent of reference mesh.py:79-107."""
    tri = np.asarray(mesh.triangles, dtype=np.int64)
    E = len(tri)
    nv = max(int(tri.max()) + 1 if E else 0, mesh.n_vertices)
    u = np.stack([tri[:, a] for a, _ in _LOCAL], axis=1).ravel()  # flat t*3+j
    v = np.stack([tri[:, b] for _, b in _LOCAL], axis=1).ravel()
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    key = lo * nv + hi
    order = np.argsort(key, kind="stable")
    skey = key[order]
    starts = np.flatnonzero(np.r_[True, skey[1:] != skey[:-1]]) if E else np.zeros(0, np.int64)
    counts = np.diff(np.r_[starts, len(skey)])
    if (counts > 2).any():
        bad = int(skey[starts[np.argmax(counts > 2)]])
        raise ConnectivityError(f"edge {(bad // nv, bad % nv)} shared by more than two triangles")
    first = order[starts]
    second = np.where(counts == 2, order[np.minimum(starts + 1, len(order) - 1)], -1)
    # same-direction traversal check (mesh.py:96-100)
    two = counts == 2
    same = two & (u[first] == u[np.maximum(second, 0)]) & (v[first] == v[np.maximum(second, 0)])
    if same.any():
        g = int(np.argmax(same))
        raise ConnectivityError(
            f"triangles {first[g] // 3} and {second[g] // 3} traverse edge "
            f"{(int(lo[first[g]]), int(hi[first[g]]))} in the same direction "
            "(inconsistent orientation)")
    # first-encounter order
    eo = np.argsort(first, kind="stable")
    first, second, counts = first[eo], second[eo], counts[eo]
    ne = len(first)
    left, left_local = first // 3, first % 3
    right = np.where(second >= 0, second // 3, -1)
    right_local = np.where(second >= 0, second % 3, -1)
    marker = np.zeros(ne, dtype=np.int64)
    bnd = right < 0
    marker[bnd] = DIRICHLET
    if mesh.boundary_markers:
        lut = {int(min(a, b)) * nv + int(max(a, b)): int(m)
               for (a, b), m in mesh.boundary_markers.items()}
        bk = (lo[first] * nv + hi[first])[bnd]
        marker[np.flatnonzero(bnd)] = [lut.get(int(k_), DIRICHLET) for k_ in bk]
    elem_edge = np.empty((E, 3), dtype=np.int64)
    nbr = np.full((E, 3), -1, dtype=np.int64)
    nbr_local = np.empty((E, 3), dtype=np.int64)
    idx = np.arange(ne)
    elem_edge[left, left_local] = idx
    nbr_local[left, left_local] = -marker
    it = ~bnd
    elem_edge[right[it], right_local[it]] = idx[it]
    nbr[left[it], left_local[it]] = right[it]
    nbr_local[left[it], left_local[it]] = right_local[it]
    nbr[right[it], right_local[it]] = left[it]
    nbr_local[right[it], right_local[it]] = left_local[it]
    mesh._conn = Connectivity(
        v0=u[first], v1=v[first], left=left, left_local=left_local, right=right,
        right_local=right_local, marker=marker, elem_edge=elem_edge, nbr=nbr,
        nbr_local=nbr_local)
    mesh._edges_cache = None


def _signed_dets(vertices: np.ndarray, triangles: np.ndarray) -> np.ndarray:
    a, b, c = (vertices[triangles[:, i]] for i in range(3))
    return (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (the published mixer; reference mesh.py:119-125)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def jitter_unit(seed: int, vertex_ids: np.ndarray, coord: int, retry) -> np.ndarray:
    """Uniforms in [-1, 1) keyed by (seed, vertex, coord, retry) (mesh.py:128-136)."""
    retry = np.asarray(retry, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
               ^ _splitmix64(vertex_ids.astype(np.uint64) * np.uint64(4) + np.uint64(coord))
               ^ _splitmix64(retry + np.uint64(0x5DEECE66D)))
    return _splitmix64(key).astype(np.float64) / 2.0**63 - 1.0


def _finish(vertices, triangles, markers=None, lazy: bool = False) -> Mesh:
    mesh = Mesh(vertices=vertices, triangles=triangles, boundary_markers=markers or {})
    if not lazy:
        build_connectivity(mesh)
    return mesh


def build_square_mesh(level: int, perturb: float = 0.0, seed: int = 0) -> Mesh:
    """Reference generator (mesh.py:139-196): [0,1000]^2, checkerboard split,
    every vertex jittered by perturb*h, per-vertex retries on inversion."""
    if level < 1 or level > 8:
        raise ValueError("level must be in 1..8")
    if not 0.0 <= perturb <= 0.2:
        raise ValueError("perturb must be in [0, 0.2]")
    n = 2**level
    h = 1000.0 / n
    xs = np.linspace(0.0, 1000.0, n + 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    base = np.column_stack([X.ravel(), Y.ravel()])
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    v00, v10 = i * (n + 1) + j, (i + 1) * (n + 1) + j
    v11, v01 = (i + 1) * (n + 1) + j + 1, i * (n + 1) + j + 1
    even = (i + j) % 2 == 0
    t1 = np.where(even[:, None], np.stack([v00, v10, v11], 1), np.stack([v00, v10, v01], 1))
    t2 = np.where(even[:, None], np.stack([v00, v11, v01], 1), np.stack([v10, v11, v01], 1))
    tris = np.stack([t1, t2], axis=1).reshape(-1, 3).astype(np.int64)
    verts = base.copy()
    if perturb > 0.0:
        ids = np.arange(len(base), dtype=np.uint64)
        retry = np.zeros(len(base), dtype=np.int64)
        for _ in range(100):
            for c in (0, 1):
                verts[:, c] = base[:, c] + perturb * h * jitter_unit(seed, ids, c, retry)
            bad = _signed_dets(verts, tris) <= 0.0
            if not bad.any():
                break
            retry[np.unique(tris[bad])] += 1
        else:
            raise DegenerateElement("perturbation produced a degenerate triangle after 100 retries")
    return _finish(verts, tris)


def build_unit_square_mesh(n: int, jitter: float = 0.0, seed: int = 0,
                           length: float = 1.0, lazy: bool = False) -> Mesh:
    """BASELINE mesh: [0,L]^2, n x n quads, every quad split SW-NE into
    (v00, v10, v11), (v00, v11, v01); vertex id = i*(n+1)+j (x index i).

    ``jitter`` > 0 displaces INTERIOR vertices by jitter*h*u, u in [-1, 1)
    from ``jitter_unit`` (SplitMix64 keyed by seed/vertex/coord, retry 0).
    With jitter <= 0.25 no triangle can invert (min altitude h/sqrt2).
    ``lazy``: connectivity is built on first use of ``mesh.conn`` (the device
    setup path, device_setup.py, never needs it).
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    h = length / n
    xs = np.linspace(0.0, length, n + 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    verts = np.column_stack([X.ravel(), Y.ravel()])
    i, j = np.meshgrid(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64), indexing="ij")
    i, j = i.ravel(), j.ravel()
    v00, v10 = i * (n + 1) + j, (i + 1) * (n + 1) + j
    v11, v01 = (i + 1) * (n + 1) + j + 1, i * (n + 1) + j + 1
    tris = np.stack([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)],
                    axis=1).reshape(-1, 3)
    if jitter > 0.0:
        if jitter > 0.25:
            raise ValueError("jitter must be <= 0.25 (no inversion guarantee)")
        I, Jv = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
        inner = ((I > 0) & (I < n) & (Jv > 0) & (Jv < n)).ravel()
        ids = np.flatnonzero(inner).astype(np.uint64)
        for c in (0, 1):
            verts[inner, c] += jitter * h * jitter_unit(seed, ids, c, 0)
        if (_signed_dets(verts, tris) <= 0.0).any():
            raise DegenerateElement("jitter inverted a triangle")
    return _finish(verts, tris, lazy=lazy)


def build_ring_mesh(level: int) -> Mesh:
    """Annulus 500 <= r <= 1000 from 8*(2^level)^2 split quads (mesh.py:199-238)."""
    if level < 1 or level > 8:
        raise ValueError("level must be in 1..8")
    n = 2**level
    n_ang, n_rad = 8 * n, n
    thetas = np.linspace(0.0, 2.0 * np.pi, n_ang, endpoint=False)
    radii = np.linspace(500.0, 1000.0, n_rad + 1)
    A, Rr = np.meshgrid(np.arange(n_ang), np.arange(n_rad + 1), indexing="ij")
    verts = np.column_stack([(radii[Rr] * np.cos(thetas[A])).ravel(),
                             (radii[Rr] * np.sin(thetas[A])).ravel()])

    def vid(a, ri):
        return (a % n_ang) * (n_rad + 1) + ri

    a, ri = np.meshgrid(np.arange(n_ang), np.arange(n_rad), indexing="ij")
    a, ri = a.ravel(), ri.ravel()
    p1, p2, p3, p4 = vid(a, ri), vid(a, ri + 1), vid(a + 1, ri + 1), vid(a + 1, ri)
    even = (a + ri) % 2 == 0
    t1 = np.where(even[:, None], np.stack([p1, p2, p3], 1), np.stack([p1, p2, p4], 1))
    t2 = np.where(even[:, None], np.stack([p1, p3, p4], 1), np.stack([p2, p3, p4], 1))
    tris = np.stack([t1, t2], axis=1).reshape(-1, 3).astype(np.int64)
    return _finish(verts, tris)


@dataclass
class ElementGeometry:
    B: np.ndarray          # (E, 2, 2), columns a2-a1, a3-a1
    detB: np.ndarray       # (E,)
    sqrt_detB: np.ndarray  # (E,)
    a1: np.ndarray         # (E, 2)


@dataclass
class EdgeGeometry:
    normal: np.ndarray     # (NE, 2) outward unit normal of the left triangle
    length: np.ndarray     # (NE,)


def compute_geometry(mesh: Mesh) -> tuple[ElementGeometry, EdgeGeometry]:
    """Vectorised reference mesh.py:259-282."""
    v, t = mesh.vertices, mesh.triangles
    a1 = v[t[:, 0]]
    B = np.stack([v[t[:, 1]] - a1, v[t[:, 2]] - a1], axis=2)
    detB = B[:, 0, 0] * B[:, 1, 1] - B[:, 0, 1] * B[:, 1, 0]
    if (detB <= 0.0).any():
        bad = int(np.argmax(detB <= 0.0))
        raise DegenerateElement(f"triangle {bad} has detB = {detB[bad]:.3e}")
    c = mesh.conn
    d = v[c.v1] - v[c.v0]
    length = np.hypot(d[:, 0], d[:, 1])
    normal = np.column_stack([d[:, 1] / length, -d[:, 0] / length])
    return (ElementGeometry(B=B, detB=detB, sqrt_detB=np.sqrt(detB), a1=a1),
            EdgeGeometry(normal=normal, length=length))


def save_mesh(mesh: Mesh, path) -> None:
    """``ghoddess-mesh 1`` text format (reference mesh.py:288-301)."""
    c = mesh.conn
    lines = [FORMAT_HEADER, f"vertices {mesh.n_vertices}"]
    lines += [f"{x:.17g} {y:.17g}" for x, y in mesh.vertices]
    lines.append(f"triangles {mesh.n_triangles}")
    lines += [f"{a} {b} {cc}" for a, b, cc in mesh.triangles]
    bnd = np.flatnonzero(c.right < 0)
    lines.append(f"boundary {len(bnd)}")
    lines += [f"{c.v0[i]} {c.v1[i]} {c.marker[i]}" for i in bnd]
    Path(path).write_text("\n".join(lines) + "\n")


def load_mesh(path) -> Mesh:
    """Parse ``ghoddess-mesh 1`` (reference mesh.py:304-373); errors carry line numbers."""
    raw = Path(path).read_text().splitlines()
    rows = [(no + 1, line.split("#", 1)[0].strip()) for no, line in enumerate(raw)]
    rows = [(no, text) for no, text in rows if text]
    pos = 0

    def take():
        nonlocal pos
        if pos >= len(rows):
            raise MeshParseError(f"line {len(raw)}: unexpected end of file")
        pos += 1
        return rows[pos - 1]

    no, text = take()
    if text != FORMAT_HEADER:
        raise MeshParseError(f"line {no}: expected header {FORMAT_HEADER!r}")

    def section(keyword):
        no, text = take()
        parts = text.split()
        if len(parts) != 2 or parts[0] != keyword or not parts[1].isdigit():
            raise MeshParseError(f"line {no}: expected '{keyword} <count>'")
        return int(parts[1])

    nv = section("vertices")
    verts = np.empty((nv, 2))
    for i in range(nv):
        no, text = take()
        parts = text.split()
        try:
            if len(parts) != 2:
                raise ValueError
            verts[i] = (float(parts[0]), float(parts[1]))
        except ValueError:
            raise MeshParseError(f"line {no}: expected 'x y'") from None
    nt = section("triangles")
    tris = np.empty((nt, 3), dtype=np.int64)
    for i in range(nt):
        no, text = take()
        parts = text.split()
        try:
            if len(parts) != 3:
                raise ValueError
            tris[i] = [int(p) for p in parts]
        except ValueError:
            raise MeshParseError(f"line {no}: expected 'v0 v1 v2'") from None
        if (tris[i] < 0).any() or (tris[i] >= nv).any():
            raise MeshParseError(f"line {no}: vertex index out of range")
    nb = section("boundary")
    markers = {}
    for _ in range(nb):
        no, text = take()
        parts = text.split()
        try:
            if len(parts) != 3:
                raise ValueError
            a, b, m = (int(p) for p in parts)
        except ValueError:
            raise MeshParseError(f"line {no}: expected 'v0 v1 marker'") from None
        if not (0 <= a < nv and 0 <= b < nv):
            raise MeshParseError(f"line {no}: vertex index out of range")
        markers[(min(a, b), max(a, b))] = m
    return _finish(verts, tris, markers)


def _spread16(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0xFFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
    return v


def locality_order(mesh: Mesh, elements=None) -> np.ndarray:
    """Z-order (Morton) permutation of ``elements`` by centroid.

    Consecutive runs of the result are compact patches of the mesh, so a
    thread block of the stage kernel finds most neighbours of its elements
    inside the block (shared-memory trace exchange instead of global
    gathers).  Returns positions into ``elements`` (default: all).
    """
    el = np.arange(mesh.n_triangles) if elements is None else np.asarray(elements)
    if len(el) == 0:
        return np.zeros(0, dtype=np.int64)
    cen = mesh.vertices[mesh.triangles[el]].mean(axis=1)
    lo, hi = cen.min(axis=0), cen.max(axis=0)
    # lattice of the element size (sqrt of twice the mean area: the quad
    # side of a split-square mesh, whose two triangles then share a cell), so
    # that aligned Morton blocks are whole square patches for any N, not
    # only powers of two (N = 1448: 28 -> 54 out-of-block edges per
    # 128-element block with the range-scaled lattice)
    v = mesh.vertices[mesh.triangles[el]]
    area = 0.5 * np.abs((v[:, 1, 0] - v[:, 0, 0]) * (v[:, 2, 1] - v[:, 0, 1])
                        - (v[:, 2, 0] - v[:, 0, 0]) * (v[:, 1, 1] - v[:, 0, 1]))
    h = float(np.sqrt(2.0 * area.mean()))
    span = float((hi - lo).max())
    if h > 0.0 and span / h < 65535.0:
        q = np.floor((cen - lo) / h + 1.0 / 6.0).astype(np.int64)
    else:
        q = ((cen - lo) / np.maximum(hi - lo, 1e-300) * 65535.0).astype(np.int64)
    code = _spread16(q[:, 0]) | (_spread16(q[:, 1]) << np.uint64(1))
    return np.argsort(code, kind="stable")
