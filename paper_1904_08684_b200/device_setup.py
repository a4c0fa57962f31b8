"""Device-side mesh setup: geometry, connectivity, Z-order
slots and the SoA element tables built on the GPU.

The host path (``mesh.build_connectivity``, ``mesh.compute_geometry``,
``mesh.locality_order``, ``layout.build_tables``: vectorised NumPy
restatements of reference mesh.py:79-107, 259-282) takes about a minute at
the BASELINE C5 strong-scaling size (2 x 4096^2 = 33.5M triangles).  Here
the same algorithm runs as device tensor operations:

* connectivity: every (triangle, local edge j) yields the key
  min(v) * NV + max(v) of its vertex pair (local edge j = (a_{j+1},
  a_{j+2}), reference mesh.py:84); a stable device sort puts the two
  occurrences of an interior edge next to each other, which gives each
  element's neighbour and the neighbour's local edge; an unmatched key is a
  boundary edge (its marker from ``mesh.boundary_markers``, default
  Dirichlet = 1, looked up on the host for the O(sqrt E) boundary edges);
* geometry: B = [a2 - a1, a3 - a1], det B, edge lengths, h_min =
  min(det B / longest edge) (reference solver.py:240-246);
* slots: the Morton code of each centroid on the element-size lattice, the
  same integer code as ``mesh.locality_order``, sorted on the device;
* tables: geo[6][ld] and the neighbour codes nbr[3][ld] in slot order;
  Dirichlet slots in mesh-edge (first-encounter) order, which for a
  boundary edge is the order of its flat index 3 e + j.

The results are bit-identical to the host path (``tests``: device tables ==
host tables); the host connectivity (``mesh.conn``, reference ``Edge``
list) stays available lazily for the APIs that report per mesh edge.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import BND_DIRICHLET, BND_WALL, pad_ld
from .mesh import DIRICHLET, ConnectivityError, DegenerateElement, Mesh

__all__ = ["DeviceTables", "device_tables"]


@dataclass
class DeviceTables:
    """``layout.ElementTables`` with device tensors (same meaning)."""

    n_elem: int
    ld: int
    geo: object        # torch (6, ld) float64
    nbr: object        # torch (3, ld) int32
    bnd_elem: object   # torch (nb,) int32
    bnd_local: object  # torch (nb,) int32
    h_min: float
    perm: object       # torch (E,) int64: slot -> mesh element
    seconds: float = 0.0

    def host(self, name):
        return getattr(self, name).cpu().numpy()


def _spread16(v):
    v = v & 0xFFFF
    v = (v | (v << 8)) & 0x00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333
    v = (v | (v << 1)) & 0x55555555
    return v


def device_tables(mesh: Mesh, dirichlet_markers, wall_markers, device) -> DeviceTables:
    """Element tables of a whole mesh in Z-order slots, built on ``device``."""
    import time

    import torch

    t0 = time.perf_counter()
    dev = torch.device(device)
    V = torch.as_tensor(np.ascontiguousarray(mesh.vertices, dtype=np.float64), device=dev)
    T = torch.as_tensor(np.ascontiguousarray(mesh.triangles, dtype=np.int64), device=dev)
    E, nv = T.shape[0], V.shape[0]
    if E == 0:
        raise ValueError("empty mesh")
    # ---- geometry (reference mesh.py:259-282)
    a1 = V[T[:, 0]]
    b1, b2 = V[T[:, 1]] - a1, V[T[:, 2]] - a1
    B11, B21, B12, B22 = b1[:, 0], b1[:, 1], b2[:, 0], b2[:, 1]
    det = B11 * B22 - B12 * B21
    if bool((det <= 0.0).any()):
        bad = int(torch.argmax((det <= 0.0).to(torch.int8)))
        raise DegenerateElement(f"triangle {bad} has detB = {float(det[bad]):.3e}")
    # ---- connectivity (reference mesh.py:79-107): flat f = 3 e + j
    u = T[:, [1, 2, 0]].reshape(-1)
    v = T[:, [2, 0, 1]].reshape(-1)
    lo, hi = torch.minimum(u, v), torch.maximum(u, v)
    key = lo * nv + hi
    skey, order = torch.sort(key, stable=True)
    same = skey[1:] == skey[:-1]
    if E >= 1 and len(skey) > 2 and bool((same[1:] & same[:-1]).any()):
        raise ConnectivityError("an edge is shared by more than two triangles")
    i = torch.nonzero(same).squeeze(1)
    fa, fb = order[i], order[i + 1]
    if bool(((u[fa] == u[fb]) & (v[fa] == v[fb])).any()):
        raise ConnectivityError("two triangles traverse an edge in the same direction "
                                "(inconsistent orientation)")
    nbr = torch.full((3 * E,), -1, dtype=torch.int64, device=dev)
    nloc = torch.full((3 * E,), -1, dtype=torch.int64, device=dev)
    nbr[fa], nloc[fa] = fb // 3, fb % 3
    nbr[fb], nloc[fb] = fa // 3, fa % 3
    bflat = torch.nonzero(nbr < 0).squeeze(1)  # boundary (e, j), ascending 3 e + j
    # boundary markers on the host (O(sqrt E) edges)
    mk = np.full(len(bflat), DIRICHLET, dtype=np.int64)
    if mesh.boundary_markers:
        bk = key[bflat].cpu().numpy()
        lut = {int(min(a, b)) * nv + int(max(a, b)): int(m)
               for (a, b), m in mesh.boundary_markers.items()}
        mk = np.array([lut.get(int(k_), DIRICHLET) for k_ in bk], dtype=np.int64)
    dmask = np.isin(mk, list(dirichlet_markers))
    wmask = np.isin(mk, list(wall_markers))
    if not (dmask | wmask).all():
        bad = int(np.flatnonzero(~(dmask | wmask))[0])
        raise ValueError(f"boundary edge of element {int(bflat[bad]) // 3} has marker "
                         f"{mk[bad]}; only Dirichlet and wall markers are supported")
    # ---- h_min = min(detB / longest edge) (solver.py:240-246)
    # (device hypot may differ from libm's in the last ulp: the few candidate
    # minimisers are re-evaluated on the host with the host path's formula)
    d = V[v] - V[u]
    ratio = det / torch.hypot(d[:, 0], d[:, 1]).view(E, 3).max(dim=1).values
    cand = torch.nonzero(ratio <= ratio.min() * (1.0 + 1e-12)).squeeze(1).cpu().numpy()
    tri = np.asarray(mesh.triangles)[cand]
    vv = np.asarray(mesh.vertices, dtype=np.float64)
    ca1, cb1, cb2 = vv[tri[:, 0]], vv[tri[:, 1]] - vv[tri[:, 0]], vv[tri[:, 2]] - vv[tri[:, 0]]
    cdet = cb1[:, 0] * cb2[:, 1] - cb2[:, 0] * cb1[:, 1]
    lens = np.stack([np.hypot(*(vv[tri[:, b]] - vv[tri[:, a]]).T)
                     for a, b in ((1, 2), (2, 0), (0, 1))], axis=1)
    h_min = float((cdet / lens.max(axis=1)).min())
    del ca1
    # ---- Z-order slots (mesh.locality_order, same integer codes)
    # (host: vertices[triangles].mean(axis=1) = ((a + b) + c) / 3)
    cen = ((V[T[:, 0]] + V[T[:, 1]]) + V[T[:, 2]]) / 3.0
    clo, chi = cen.min(dim=0).values, cen.max(dim=0).values
    area = 0.5 * torch.abs((b1[:, 0] * b2[:, 1]) - (b2[:, 0] * b1[:, 1]))
    h = float(torch.sqrt(2.0 * area.mean()))
    span = float((chi - clo).max())
    if h > 0.0 and span / h < 65535.0:
        q = torch.floor((cen - clo) / h + 1.0 / 6.0).to(torch.int64)
    else:
        q = ((cen - clo) / torch.clamp(chi - clo, min=1e-300) * 65535.0).to(torch.int64)
    code = _spread16(q[:, 0]) | (_spread16(q[:, 1]) << 1)
    _, perm = torch.sort(code, stable=True)
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(E, device=dev)
    # ---- tables in slot order
    ld = pad_ld(E)
    geo = torch.zeros((6, ld), dtype=torch.float64, device=dev)
    for r, x in enumerate((B11, B12, B21, B22, a1[:, 0], a1[:, 1])):
        geo[r, :E] = x[perm]
    nb3, nl3 = nbr.view(E, 3)[perm], nloc.view(E, 3)[perm]  # (slot, j)
    codes = torch.where(nb3 >= 0, 4 * inv[torch.clamp(nb3, min=0)] + torch.clamp(nl3, min=0),
                        torch.zeros_like(nb3))
    # boundary codes: Dirichlet slot s in flat-index order, walls -1 - 1
    dm = torch.as_tensor(dmask, device=dev)
    dslot = torch.cumsum(dm.to(torch.int64), 0) - 1
    bcode = torch.where(dm, -1 - (2 * dslot + BND_DIRICHLET),
                        torch.full_like(dslot, -1 - BND_WALL))
    be, bj = bflat // 3, bflat % 3
    codes[inv[be], bj] = bcode
    nbr_t = torch.zeros((3, ld), dtype=torch.int32, device=dev)
    nbr_t[:, :E] = codes.t().to(torch.int32)
    if E and int(codes.max()) >= 2**31:
        raise ValueError("mesh too large for int32 neighbour codes")
    bel = inv[be[dm]].to(torch.int32)
    blc = bj[dm].to(torch.int32)
    torch.cuda.synchronize(dev)
    return DeviceTables(n_elem=E, ld=ld, geo=geo, nbr=nbr_t, bnd_elem=bel, bnd_local=blc,
                        h_min=h_min, perm=perm, seconds=time.perf_counter() - t0)
