"""Device data layout: structure-of-arrays element tables (host-side build).

Everything the stage kernels read is laid out field-major with the element
index fastest, so a warp of 32 consecutive elements reads one 256-byte line
per (field, mode):

    state c   [3][K][ld]   (xi, U, V) modal coefficients
    velocity  [2][K][ld]   (u, v)
    geo       [6][ld]      B11, B12, B21, B22, a1x, a1y
    hb        [NH][ld]     projected bathymetry coefficients (NH = 1 or 3)
    nbr       [3][ld]      int32 neighbour code per local edge:
                             >= 0 : 4 * neighbour + neighbour's local edge,
                                    or 4 * h + 3: row h of the halo trace
                                    table (partitions, distributed.py)
                             <  0 : boundary, -1 - (2 * slot + kind),
                                    kind 0 = Dirichlet (slot indexes the
                                    per-stage ghost table), 1 = wall
    bnd       [nb]         (element, local edge) of each Dirichlet slot

``ld`` = element count rounded up to a multiple of 32 (alignment of every
row to 256 B).  Elements [E, ld) are padding and never touched; a
partition holds only its owned elements (see ``distributed.py``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import Mesh, compute_geometry

__all__ = ["ElementTables", "build_tables", "pad_ld", "aos_to_soa", "soa_to_aos"]

BND_DIRICHLET, BND_WALL = 0, 1
HALO_J = 3  # neighbour code 4 h + 3: row h of the halo trace table (csrc HALO_J)


def pad_ld(n: int) -> int:
    return max(32, (n + 31) // 32 * 32)


@dataclass
class ElementTables:
    n_elem: int
    ld: int
    geo: np.ndarray       # (6, ld) float64
    nbr: np.ndarray       # (3, ld) int32
    bnd_elem: np.ndarray  # (nb,) int32
    bnd_local: np.ndarray  # (nb,) int32
    detB: np.ndarray      # (E,)
    h_min: float


def build_tables(mesh: Mesh, dirichlet_markers, wall_markers, elements=None, n_own=None,
                 halo_code=None) -> ElementTables:
    """Geometry and neighbour codes.

    ``elements`` (global ids, local order) restricts the tables to a
    partition: the first ``n_own`` are updated by this context.  A neighbour
    outside ``elements`` is another partition's element whose edge traces
    arrive in row h = ``halo_code[j][slot]`` of the halo trace table: code
    4 h + 3 (``HALO_J``).
    """
    geom, egeom = compute_geometry(mesh)
    c = mesh.conn
    if elements is None:
        elements = np.arange(mesh.n_triangles)
    elements = np.asarray(elements, dtype=np.int64)
    n_loc = len(elements)
    E = n_loc if n_own is None else int(n_own)
    own = elements[:E]
    ld = pad_ld(n_loc)
    g2l = np.full(mesh.n_triangles, -1, dtype=np.int64)
    g2l[elements] = np.arange(n_loc)
    geo = np.zeros((6, ld))
    B, a1 = geom.B[elements], geom.a1[elements]
    geo[0, :n_loc], geo[1, :n_loc] = B[:, 0, 0], B[:, 0, 1]
    geo[2, :n_loc], geo[3, :n_loc] = B[:, 1, 0], B[:, 1, 1]
    geo[4, :n_loc], geo[5, :n_loc] = a1[:, 0], a1[:, 1]
    nbr, nloc = c.nbr[own], c.nbr_local[own]
    inner = nbr >= 0
    lnb = np.where(inner, g2l[np.maximum(nbr, 0)], 0)
    code = np.zeros((3, ld), dtype=np.int64)
    code[:, :E] = np.where(inner, 4 * lnb + np.maximum(nloc, 0), 0).T
    ext = inner & (lnb < 0)  # neighbour owned by another partition
    if ext.any():
        if halo_code is None:
            raise ValueError("partition has remote neighbours but no halo trace rows")
        hc = np.asarray(halo_code)[:, :E].T  # (E, 3)
        if (hc[ext] < 0).any():
            raise ValueError("a remote neighbour has no halo trace row")
        ce = code[:, :E].T.copy()
        ce[ext] = 4 * hc[ext] + HALO_J
        code[:, :E] = ce.T
    bel, bj = np.nonzero(~inner)
    marks = -nloc[bel, bj]
    dmask = np.isin(marks, list(dirichlet_markers))
    wmask = np.isin(marks, list(wall_markers))
    if not (dmask | wmask).all():
        bad = int(np.flatnonzero(~(dmask | wmask))[0])
        raise ValueError(f"boundary edge of element {own[bel[bad]]} has marker {marks[bad]}; "
                         "only Dirichlet and wall markers are supported")
    # Dirichlet slots in mesh-edge order (reference pass_B order, solver.py:213-216)
    eidx = c.elem_edge[own[bel], bj]
    order = np.argsort(eidx, kind="stable")
    bel, bj, dmask = bel[order], bj[order], dmask[order]
    slot = np.cumsum(dmask) - 1
    code[bj, bel] = np.where(dmask, -1 - (2 * slot + BND_DIRICHLET), -1 - BND_WALL)
    if E and code.max() >= 2**31:
        raise ValueError("mesh too large for int32 neighbour codes")
    # CFL height (solver.py:240-246) over the owned elements
    lens = egeom.length[c.elem_edge[own]]
    h_min = float((geom.detB[own] / lens.max(axis=1)).min()) if E else float("inf")
    return ElementTables(n_elem=E, ld=ld, geo=geo, nbr=code.astype(np.int32),
                         bnd_elem=bel[dmask].astype(np.int32),
                         bnd_local=bj[dmask].astype(np.int32), detB=geom.detB[elements],
                         h_min=h_min)


def aos_to_soa(a: np.ndarray, ld: int) -> np.ndarray:
    """(E, F, K) -> (F, K, ld) with zero padding."""
    E, F, K = a.shape
    out = np.zeros((F, K, ld))
    out[:, :, :E] = a.transpose(1, 2, 0)
    return out


def soa_to_aos(s: np.ndarray, E: int) -> np.ndarray:
    return np.ascontiguousarray(s[:, :, :E].transpose(2, 0, 1))
