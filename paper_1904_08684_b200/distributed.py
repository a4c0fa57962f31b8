"""Multi-GPU: contiguous element blocks with a face-neighbour halo per stage.

The grid shards naturally: each rank owns a block of elements
(vertical strips of quad columns, or px x py rectangles on the unit-square
meshes), stores copies of the neighbour-rank elements that share an edge
with its own (the halo) after its owned elements, and after every RK stage
sends the new (c, u) of its cut-adjacent elements to the ranks that hold
them as halo.  No per-stage collective exists: lambda is per edge and dt is
fixed; one allreduce(max) fixes a CFL dt and one allreduce(max) takes the
step time.

Overlap: owned elements are ordered interior-first; per stage the interior
range runs on the compute stream while the previous stage's halo is still in
flight, then the cut-adjacent range runs once the halo has arrived, and its
result is gathered and exchanged on a communication stream while the next
stage's interior range computes.

The host logic (partitioning, halo lists, exchange) is shared by the GPU
runner (NCCL over NVLink, ``qf_stage`` / ``qf_gather`` / ``qf_scatter``) and
a CPU runner used by the ``gloo`` tests, whose stage executor is the
test-only oracle (``oracle/trace_stage.py``).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh

__all__ = ["strip_partition", "block_partition", "block_shape", "range_partition", "Halo",
           "build_halo",
           "HaloExchange", "push_table", "DistributedRunner", "bench_distributed"]


# --------------------------------------------------------------- partitions
def strip_partition(n: int, world: int) -> np.ndarray:
    """Unit-square split mesh (build_unit_square_mesh(n)): strips of quad columns."""
    q = np.arange(2 * n * n) // 2
    col = q // n
    return (col * world // n).astype(np.int64)


def block_partition(n: int, px: int, py: int) -> np.ndarray:
    """px x py rectangles of quads (C4: 4 x 2)."""
    q = np.arange(2 * n * n) // 2
    i, j = q // n, q % n
    return ((i * px // n) * py + (j * py // n)).astype(np.int64)


def range_partition(n_elem: int, world: int) -> np.ndarray:
    """Generic meshes: contiguous element ranges of equal size."""
    return (np.arange(n_elem) * world // max(n_elem, 1)).astype(np.int64)


@dataclass
class Halo:
    """Local element order and exchange lists of one rank."""

    rank: int
    elements: np.ndarray          # global ids: owned (interior, then cut-adjacent), halo
    n_own: int
    n_int: int                    # owned elements without a remote neighbour
    send: dict = field(default_factory=dict)   # peer -> local ids (owned), peer's halo order
    recv: dict = field(default_factory=dict)   # peer -> local ids (halo)

    @property
    def n_local(self) -> int:
        return len(self.elements)


def build_halo(mesh: Mesh, part: np.ndarray, rank: int) -> Halo:
    nbr = mesh.conn.nbr
    own = np.flatnonzero(part == rank)
    nb = nbr[own]
    remote = (nb >= 0) & (part[np.maximum(nb, 0)] != rank)
    cut = remote.any(axis=1)
    from .mesh import locality_order

    oi, ob = own[~cut], own[cut]
    own_order = np.concatenate([oi[locality_order(mesh, oi)], ob[locality_order(mesh, ob)]])
    n_own, n_int = len(own), int((~cut).sum())
    rem = np.unique(nb[remote])
    owner = part[rem]
    order = np.lexsort((rem, owner))
    halo = rem[order]
    elements = np.concatenate([own_order, halo])
    g2l = {int(g): i for i, g in enumerate(elements)}
    recv, send = {}, {}
    for p in np.unique(owner):
        hp = halo[owner[order] == p]
        recv[int(p)] = np.array([g2l[int(g)] for g in hp], dtype=np.int64)
        # my owned elements adjacent to p, in global-id order (= p's halo order)
        nbp = nbr[own_order]
        mine = own_order[((nbp >= 0) & (part[np.maximum(nbp, 0)] == p)).any(axis=1)]
        mine = np.sort(mine)
        send[int(p)] = np.array([g2l[int(g)] for g in mine], dtype=np.int64)
    return Halo(rank=rank, elements=elements, n_own=n_own, n_int=n_int, send=send, recv=recv)


PUSH_SLOT_BITS = 26


def push_table(halo: Halo, peer_recv: dict, ld: int) -> np.ndarray:
    """Destinations of the fused halo push (``qf_stage_push``): int32 [3][ld],
    entry (peer << 26) | slot in the peer's local order, -1 = none.

    ``peer_recv[p]`` is peer p's ``halo.recv[my rank]``: its halo slots of my
    elements, in the same (global-id) order as my ``halo.send[p]``.  An
    element adjacent to several peers gets one entry per peer (at most 3:
    one per edge)."""
    tab = np.full((3, ld), -1, dtype=np.int32)
    fill = np.zeros(ld, dtype=np.int64)
    for p, mine in halo.send.items():
        dst = np.asarray(peer_recv[p], dtype=np.int64)
        if len(dst) != len(mine):
            raise ValueError(f"halo lists of rank {halo.rank} and peer {p} disagree")
        if p >= 1 << (31 - PUSH_SLOT_BITS) or (len(dst) and dst.max() >= 1 << PUSH_SLOT_BITS):
            raise ValueError("push table overflow (peer or slot index)")
        for e, d in zip(np.asarray(mine, dtype=np.int64), dst):
            tab[fill[e], e] = (p << PUSH_SLOT_BITS) | int(d)
            fill[e] += 1
    return tab


def peer_table(torch, entries, device):
    """Device qf_peer[] table: entries[p] = (c_ptr, u_ptr, ld) or None."""
    t = torch.zeros((max(len(entries), 1), 3), dtype=torch.int64)
    for p, ent in enumerate(entries):
        if ent is not None:
            t[p, 0], t[p, 1], t[p, 2] = int(ent[0]), int(ent[1]), int(ent[2])
    return t.to(device)


# ----------------------------------------------------------------- exchange
class HaloExchange:
    """Pack (c, u) rows of the send lists, P2P exchange, unpack into the halo.

    ``c``/``u`` are [F][K][ld] tensors (device for NCCL, CPU for gloo).  On
    the GPU, gather/scatter are the library kernels; the transfers are
    ``torch.distributed.batch_isend_irecv`` (NCCL P2P over NVLink).
    """

    def __init__(self, halo: Halo, K: int, ld: int, device, lib=None):
        import torch

        self.torch = torch
        self.halo, self.K, self.ld, self.lib = halo, K, ld, lib
        self.rows = 5 * K
        self.dev = device
        self.peers = sorted(set(halo.send) | set(halo.recv))
        self.sidx = {p: torch.as_tensor(halo.send.get(p, np.zeros(0, np.int64)).astype(np.int32),
                                        device=device) for p in self.peers}
        self.ridx = {p: torch.as_tensor(halo.recv.get(p, np.zeros(0, np.int64)).astype(np.int32),
                                        device=device) for p in self.peers}
        self.sbuf = {p: torch.empty(self.rows * len(self.sidx[p]), dtype=torch.float64,
                                    device=device) for p in self.peers}
        self.rbuf = {p: torch.empty(self.rows * len(self.ridx[p]), dtype=torch.float64,
                                    device=device) for p in self.peers}

    def _gather(self, c, u, p, stream):
        n = len(self.sidx[p])
        buf = self.sbuf[p]
        if self.lib is not None:
            s = stream.cuda_stream
            self.lib.qf_gather(c.data_ptr(), self.ld, self.sidx[p].data_ptr(), n, 3 * self.K,
                               buf.data_ptr(), s)
            self.lib.qf_gather(u.data_ptr(), self.ld, self.sidx[p].data_ptr(), n, 2 * self.K,
                               buf[3 * self.K * n:].data_ptr(), s)
        else:
            idx = self.sidx[p].long()
            buf.view(self.rows, n)[: 3 * self.K] = c.view(3 * self.K, self.ld)[:, idx]
            buf.view(self.rows, n)[3 * self.K:] = u.view(2 * self.K, self.ld)[:, idx]

    def _scatter(self, c, u, p, stream):
        n = len(self.ridx[p])
        buf = self.rbuf[p]
        if self.lib is not None:
            s = stream.cuda_stream
            self.lib.qf_scatter(buf.data_ptr(), self.ridx[p].data_ptr(), n, 3 * self.K,
                                c.data_ptr(), self.ld, s)
            self.lib.qf_scatter(buf[3 * self.K * n:].data_ptr(), self.ridx[p].data_ptr(), n,
                                2 * self.K, u.data_ptr(), self.ld, s)
        else:
            idx = self.ridx[p].long()
            c.view(3 * self.K, self.ld)[:, idx] = buf.view(self.rows, n)[: 3 * self.K]
            u.view(2 * self.K, self.ld)[:, idx] = buf.view(self.rows, n)[3 * self.K:]

    def exchange(self, c, u, stream=None):
        """Blocking (w.r.t. ``stream``) halo update of (c, u)."""
        import torch.distributed as dist

        for p in self.peers:
            self._gather(c, u, p, stream)
        ops = []
        for p in self.peers:
            if len(self.sbuf[p]):
                ops.append(dist.P2POp(dist.isend, self.sbuf[p], p))
            if len(self.rbuf[p]):
                ops.append(dist.P2POp(dist.irecv, self.rbuf[p], p))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for p in self.peers:
            self._scatter(c, u, p, stream)


def rk_plan(k: int):
    """(src, dst, a, b, toff) per stage over buffers 0 (state), 1, 2."""
    if k == 0:
        return [(0, 1, 0.0, 1.0, 0.0)]
    if k == 1:
        return [(0, 1, 0.0, 1.0, 0.0), (1, 0, 0.5, 0.5, 1.0)]
    return [(0, 1, 0.0, 1.0, 0.0), (1, 2, 0.75, 0.25, 1.0), (2, 0, 1.0 / 3.0, 2.0 / 3.0, 0.5)]


# ------------------------------------------------------------- GPU runner
class PartitionRunner:
    """Device state and stage launches of one partition (owned + halo)."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray, rank: int):
        import torch

        from .solver import Discretization

        self.torch = torch
        self.k = order
        self.halo = build_halo(mesh, part, rank)
        h = self.halo
        self.disc = Discretization(mesh, scenario, order, elements=h.elements, n_own=h.n_own)
        d = self.disc
        self.K, self.ld, self.lib = d.K, d.ld, d._lib
        self.c = d._c_init.clone() if d.device_setup else d.upload_fields(d.project_fields())
        self.u = torch.zeros_like(self.c[:2])
        self.bufs = {0: (self.c, self.u),
                     1: (torch.zeros_like(self.c), torch.zeros_like(self.u)),
                     2: (torch.zeros_like(self.c), torch.zeros_like(self.u))}
        s = torch.cuda.current_stream().cuda_stream
        # halo velocities are element-local: solve them locally at start
        d._check(self.lib.qf_velocity(d._ctx, self.c.data_ptr(), self.u.data_ptr(), 0,
                                      h.n_local, s), "qf_velocity")
        self.dt = d.dt
        self.t = 0.0

    def local_lambda_max(self) -> float:
        d, torch = self.disc, self.torch
        lam = torch.zeros((3, self.ld), dtype=torch.float64, device=d.device)
        out = torch.empty_like(self.c)
        d._check(self.lib.qf_rhs(d._ctx, self.c.data_ptr(), self.u.data_ptr(), 0.0, 2,
                                 out.data_ptr(), lam.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream), "qf_rhs")
        return float(lam[:, : self.halo.n_own].max().item())

    def ghost(self, si: int, stream):
        """Dirichlet data of stage ``si`` (read by both ranges of the stage)."""
        d = self.disc
        if d.tables.bnd_elem.size:
            self.lib.qf_ghost(d._ctx, self.t + rk_plan(self.k)[si][4] * self.dt, stream.cuda_stream)

    def stage(self, si: int, part: str, stream, ghost: bool = True, push=None, peers=None):
        """Launch stage ``si`` on the 'interior', 'boundary' or 'all' owned range
        (with ``ghost``, the interior / all launch is preceded by the stage's
        Dirichlet data).  ``push``/``peers`` (device tensors): fused halo push
        of the new cut-adjacent rows into the peers' stage-output buffers."""
        src, dst, a, b, toff = rk_plan(self.k)[si]
        d, lib, h = self.disc, self.lib, self.halo
        s = stream.cuda_stream
        ts = self.t + toff * self.dt
        if ghost and part in ("interior", "all"):
            self.ghost(si, stream)
        ci, ui = self.bufs[src]
        co, uo = self.bufs[dst]
        e0, n = {"interior": (0, h.n_int), "boundary": (h.n_int, h.n_own - h.n_int),
                 "all": (0, h.n_own)}[part]
        if n > 0 and push is not None:
            d._check(lib.qf_stage_push(d._ctx, ci.data_ptr(), ui.data_ptr(), self.c.data_ptr(),
                                       co.data_ptr(), uo.data_ptr(), a, b, ts, self.dt, None,
                                       0.0, e0, n, push.data_ptr(), peers.data_ptr(), s),
                     "qf_stage_push")
        elif n > 0:
            d._check(lib.qf_stage(d._ctx, ci.data_ptr(), ui.data_ptr(), self.c.data_ptr(),
                                  co.data_ptr(), uo.data_ptr(), a, b, ts, self.dt, None, 0.0, e0,
                                  n, s), "qf_stage")
        return co, uo

    def end_step(self):
        if self.k == 0:
            self.torch.cuda.current_stream().wait_stream(getattr(self, "comm", None)
                                                         or self.torch.cuda.current_stream())
            self.c.copy_(self.bufs[1][0])
            self.u.copy_(self.bufs[1][1])
        self.t += self.dt


class DistributedRunner(PartitionRunner):
    """One rank of a partitioned run (one process per GPU, NCCL P2P halos)."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray, rank: int,
                 world: int, transport: str = "nccl"):
        import torch
        import torch.distributed as dist

        super().__init__(mesh, scenario, order, part, rank)
        self.dist, self.rank, self.world = dist, rank, world
        if transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        if transport == "p2p" and order == 0:
            # (Euler copies the stage output back over the halo rows a peer may
            # still be pushing into)
            raise NotImplementedError("p2p transport needs k >= 1")
        self.transport = transport
        self.transport_note = None
        if transport == "p2p" and not self._setup_p2p(mesh, part):
            # every rank falls back together (e.g. no peer access between
            # these GPUs); recorded in the bench line
            self.transport = "nccl"
        if self.transport == "nccl":
            self.ex = HaloExchange(self.halo, self.K, self.ld, self.disc.device, lib=self.lib)
        if scenario.cfl is not None:
            lmax = torch.tensor([self.local_lambda_max()], dtype=torch.float64, device="cuda")
            hmin = torch.tensor([self.disc.h_min], dtype=torch.float64, device="cuda")
            dist.all_reduce(lmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(hmin, op=dist.ReduceOp.MIN)
            from .solver import cfl_time_step
            self.dt = cfl_time_step(scenario.cfl, order, float(hmin.item()), float(lmax.item()))
        self.comm = torch.cuda.Stream()
        self.bnd = torch.cuda.Stream()

    def _setup_p2p(self, mesh, part) -> bool:
        """Fused transport: map the peers' stage buffers (CUDA IPC over
        NVLink) and build the push table; per stage the cut-adjacent launch
        stores its new rows straight into the peers' halo slots and raises a
        per-peer flag (stream memory operation); the peer's next cut-adjacent
        launch waits on that flag (no NCCL, no gather / scatter kernels).
        Collective-safe: every rank reaches the same collectives and all
        ranks agree on the outcome (False: use NCCL)."""
        import ctypes as C

        torch, dist, lib = self.torch, self.dist, self.lib
        h = self.halo
        self.peers = sorted(set(h.send) | set(h.recv))
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=self.disc.device)
        bufs = [t for b in range(3) for t in self.bufs[b]] + [self.flags]
        mine, err = [], None
        try:
            for t in bufs:
                hd = (C.c_char * 64)()
                off = C.c_uint64(0)
                self.disc._check(lib.qf_ipc_export(t.data_ptr(), hd, C.byref(off)),
                                 "qf_ipc_export")
                mine.append((bytes(hd), int(off.value)))
        except Exception as exc:  # noqa: BLE001 (reported, all ranks fall back)
            err, mine = exc, None
        info = [None] * self.world
        dist.all_gather_object(info, {"ipc": mine, "recv": {int(p): v.tolist()
                                                            for p, v in h.recv.items()},
                                      "ld": self.ld})
        try:
            if err is not None:
                raise err
            if any(info[p]["ipc"] is None for p in self.peers):
                raise RuntimeError("a peer could not export its buffers")
            ptrs = {}
            for p in self.peers:
                got = []
                for hd, off in info[p]["ipc"]:
                    ptr = C.c_void_p()
                    self.disc._check(lib.qf_ipc_import(hd, off, C.byref(ptr)), "qf_ipc_import")
                    got.append(ptr.value)
                ptrs[p] = got
            dev = self.disc.device
            self.push = torch.as_tensor(push_table(h, {p: info[p]["recv"][self.rank]
                                                       for p in h.send}, self.ld), device=dev)
            self.peer_bufs = [peer_table(torch, [(ptrs[p][2 * b], ptrs[p][2 * b + 1],
                                                  info[p]["ld"]) if p in ptrs else None
                                                 for p in range(self.world)], dev)
                              for b in range(3)]
            # my flag slot in each peer's flag array; handshake write of 0
            self.remote_flag = {p: ptrs[p][6] + 4 * self.rank for p in self.peers}
            s = torch.cuda.current_stream().cuda_stream
            for p in self.peers:
                self.disc._check(lib.qf_signal(self.remote_flag[p], 0, s), "qf_signal")
            torch.cuda.synchronize()
            ok = 1
        except Exception as exc:  # noqa: BLE001
            self.transport_note = f"p2p unavailable on rank {self.rank}: {exc}"
            ok = 0
        st = torch.tensor([ok], dtype=torch.int32,
                          device="cpu" if dist.get_backend() == "gloo" else self.disc.device)
        dist.all_reduce(st, op=dist.ReduceOp.MIN)
        dist.barrier()
        if int(st.item()) == 0:
            if self.transport_note is None:
                self.transport_note = "p2p unavailable on another rank"
            return False
        self.gen = 0  # stages completed (flag value)
        return True

    def _step_p2p(self):
        torch, lib = self.torch, self.lib
        main = torch.cuda.current_stream()
        for si in range(len(rk_plan(self.k))):
            self.ghost(si, main)
            ready = main.record_event()
            self.stage(si, "interior", main, ghost=False)
            self.bnd.wait_event(ready)
            s = self.bnd.cuda_stream
            for p in self.peers:  # the stage input's halo rows have arrived
                self.disc._check(lib.qf_wait(self.flags[p:].data_ptr(), self.gen, s), "qf_wait")
            dst = rk_plan(self.k)[si][1]
            self.stage(si, "boundary", self.bnd, ghost=False, push=self.push,
                       peers=self.peer_bufs[dst])
            self.gen += 1
            for p in self.peers:
                self.disc._check(lib.qf_signal(self.remote_flag[p], self.gen, s), "qf_signal")
            main.wait_stream(self.bnd)
        self.end_step()

    def step(self):
        """One SSP-RK step.  Per stage: the interior range (no halo
        dependence) on the main stream, concurrently the cut-adjacent range on
        its own stream once the stage input's halo has arrived, then the halo
        exchange of the new cut-adjacent rows on the communication stream,
        overlapping the next stage's interior range.

        Ordering: boundary(s) waits for the Dirichlet data of stage s and
        every launch of stage s-1 (event on main) and for exchange(s-1) (comm);
        interior(s+1) waits for boundary(s); exchange(s) waits for boundary(s).
        The two ranges of a stage write disjoint rows and read the stage input
        and the RK base only, the exchange writes halo rows that no interior
        element reads."""
        if self.transport == "p2p":
            return self._step_p2p()
        torch = self.torch
        main = torch.cuda.current_stream()
        for si in range(len(rk_plan(self.k))):
            self.ghost(si, main)
            ready = main.record_event()              # stage s-1 complete, ghost data of s
            self.stage(si, "interior", main, ghost=False)
            self.bnd.wait_event(ready)
            self.bnd.wait_stream(self.comm)          # halo of the stage input arrived
            co, uo = self.stage(si, "boundary", self.bnd, ghost=False)
            self.comm.wait_stream(self.bnd)
            with torch.cuda.stream(self.comm):
                self.ex.exchange(co, uo, self.comm)
            main.wait_stream(self.bnd)               # next stage's interior reads these rows
        self.end_step()

    def sync(self):
        main = self.torch.cuda.current_stream()
        if self.transport == "nccl":
            main.wait_stream(self.comm)
        main.wait_stream(self.bnd)


class LocalMultiRunner:
    """All partitions in one process on one GPU, halos moved by device
    gather/scatter between the partitions' buffers (fake transport for
    single-GPU tests of the partitioned kernels)."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray,
                 transport: str = "gather"):
        import torch

        self.torch = torch
        world = int(part.max()) + 1
        self.parts = [PartitionRunner(mesh, scenario, order, part, r) for r in range(world)]
        self.k = order
        self.transport = transport
        if transport == "push":  # fused: stage kernels store into each other's halo slots
            for r, pr in enumerate(self.parts):
                recv = {p: self.parts[p].halo.recv[r] for p in pr.halo.send}
                pr.push_tab = torch.as_tensor(push_table(pr.halo, recv, pr.ld), device="cuda")
                pr.peer_bufs = [peer_table(torch, [(q.bufs[b][0].data_ptr(), q.bufs[b][1].data_ptr(),
                                                    q.ld) for q in self.parts], "cuda")
                                for b in range(3)]
        idx = lambda a: torch.as_tensor(a.astype(np.int32), device="cuda")  # noqa: E731
        self.links = []
        for r, pr in enumerate(self.parts):
            for p, recv in pr.halo.recv.items():
                send = self.parts[p].halo.send[r]
                self.links.append((r, p, idx(recv), idx(send)))

    def step(self):
        torch = self.torch
        s = torch.cuda.current_stream()
        if self.transport == "push":
            for si in range(len(rk_plan(self.k))):
                dst = rk_plan(self.k)[si][1]
                for pr in self.parts:
                    pr.stage(si, "all", s, push=pr.push_tab, peers=pr.peer_bufs[dst])
            for pr in self.parts:
                pr.end_step()
            return
        for si in range(len(rk_plan(self.k))):
            outs = [pr.stage(si, "all", s) for pr in self.parts]
            for r, p, ridx, sidx in self.links:
                dst, src = self.parts[r], self.parts[p]
                n = len(ridx)
                tmp = torch.empty(5 * dst.K * n, dtype=torch.float64, device="cuda")
                for f, (arr_src, arr_dst, rows) in enumerate(
                        ((outs[p][0], outs[r][0], 3 * dst.K), (outs[p][1], outs[r][1], 2 * dst.K))):
                    off = 0 if f == 0 else 3 * dst.K * n
                    src.lib.qf_gather(arr_src.data_ptr(), src.ld, sidx.data_ptr(), n, rows,
                                      tmp[off:].data_ptr(), s.cuda_stream)
                    dst.lib.qf_scatter(tmp[off:].data_ptr(), ridx.data_ptr(), n, rows,
                                       arr_dst.data_ptr(), dst.ld, s.cuda_stream)
        for pr in self.parts:
            pr.end_step()

    def owned_state(self):
        """(global ids, c (n, 3, K)) per partition."""
        out = []
        for pr in self.parts:
            n = pr.halo.n_own
            c = pr.c[:, :, :n].permute(2, 0, 1).cpu().numpy()
            out.append((pr.halo.elements[:n], c))
        return out


# BASELINE strong-scaling meshes (configs[2]: C3 at N = 1024; configs[4]: C5 at N = 4096)
STRONG_N = {"c3": 1024, "c5": 4096}


def block_shape(world: int) -> tuple[int, int]:
    """px x py rectangles for ``world`` ranks (C4: 8 -> 4 x 2), px >= py."""
    py = int(math.isqrt(world))
    while world % py:
        py -= 1
    return world // py, py


def bench_distributed(args, configs, metric, hooks=None):
    """Weak scaling (default: N_rank = N_base^2 elements per GPU) or strong
    scaling (``--scaling strong``: the BASELINE global mesh at every N);
    strips, or px x py blocks (``--partition blocks``; default for C4).
    ``hooks`` (from bench.py): ``clocks()`` -> NVML sampler, ``peaks()`` ->
    (HBM GB/s, source), ``alg_bytes(K, r)`` -> algorithmic bytes per element."""
    import json

    import torch
    import torch.distributed as dist

    from . import mesh as M
    from . import scenario as S

    rank, world = dist.get_rank(), dist.get_world_size()
    k, n0, scen, dt, jit, desc = configs[args.config]
    scaling = getattr(args, "scaling", "weak")
    if scaling == "strong":
        # fixed global problem at every N: C3 N = 1024, C5 N = 4096 (BASELINE), or --n
        n = args.n or STRONG_N.get(args.config, n0)
    else:
        n = int(round((args.n or n0) * math.sqrt(world)))
    mesh = M.build_unit_square_mesh(n, jitter=jit, seed=7) if jit else M.build_unit_square_mesh(n)
    scn = S.mms_scenario(dt=dt) if scen == "mms" else S.bump_scenario(seed=0, cfl=0.1)
    layout = getattr(args, "partition", None) or ("blocks" if args.config == "c4" else "strips")
    if layout == "blocks":
        px, py = block_shape(world)
        part = block_partition(n, px, py)
        playout = f"blocks {px}x{py}"
    else:
        part = strip_partition(n, world)
        playout = f"strips x{world}"
    transport = getattr(args, "transport", "nccl")
    run = DistributedRunner(mesh, scn, k, part, rank, world, transport=transport)
    for _ in range(args.warmup):
        run.step()
    run.sync()
    torch.cuda.synchronize()
    dist.barrier()
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 256 MB > L2
    n_launch0 = run.lib.qf_launch_count()
    main = torch.cuda.current_stream()
    clocks = hooks["clocks"]() if hooks else None
    total = 0.0
    for it in range(args.steps):
        flush.fill_(float(it))  # outside the timed events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        run.step()
        run.sync()
        e1.record(main)
        if clocks is not None:
            clocks.sample()
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
    launches = run.lib.qf_launch_count() - n_launch0
    clk = clocks.stop() if clocks is not None else None
    # e2e: owned state H2D from pinned host memory + step + D2H of (c, u), per step
    nown, ldl = run.halo.n_own, run.ld
    host_c = torch.empty((3 * run.K, nown), dtype=torch.float64).pin_memory()
    host_cu = torch.empty((5 * run.K, nown), dtype=torch.float64).pin_memory()
    host_c.copy_(run.c.view(3 * run.K, ldl)[:, :nown].cpu())
    e2e_ms = 0.0
    n_e2e = max(3, min(args.steps, 20))
    for _ in range(n_e2e):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        run.c.view(3 * run.K, ldl)[:, :nown].copy_(host_c, non_blocking=True)
        run.step()
        run.sync()
        host_cu[: 3 * run.K].copy_(run.c.view(3 * run.K, ldl)[:, :nown], non_blocking=True)
        host_cu[3 * run.K:].copy_(run.u.view(2 * run.K, ldl)[:, :nown], non_blocking=True)
        e1.record(main)
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    ms = torch.tensor([total, e2e_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dist.barrier()
    ns = 1 if k == 0 else (2 if k == 1 else 3)
    K = run.K
    dof = 3 * K * mesh.n_triangles * ns * args.steps
    t_ms = float(ms[0].item())
    e2e_t = float(ms[1].item())
    if rank == 0:
        line = {"metric": metric, "value": dof / (t_ms * 1e-3), "unit": "DoF-updates/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc + (f" strong (fixed N={n})" if scaling == "strong"
                                               else f" weak-scaled to N={n}"),
                           "order": k, "n": n, "elements": mesh.n_triangles,
                           "parallelism": playout,
                           "halo_transport": run.transport,
                           "halo_transport_note": run.transport_note,
                           "l2": "flushed (256 MB write) between timed steps"},
                "gpu_launches": int(launches),
                "e2e": {"value": 3 * K * mesh.n_triangles * ns * n_e2e / (e2e_t * 1e-3),
                        "unit": "DoF-updates/s",
                        "h2d_bytes_per_step": 8 * 3 * K * mesh.n_triangles,
                        "d2h_bytes_per_step": 8 * 5 * K * mesh.n_triangles,
                        "timing": "per-rank owned-state H2D + step + D2H, CUDA events, max over ranks"},
                "clocks": clk}
        if hooks:
            # per GPU: algorithmic bytes of the largest rank's owned elements
            # per step over the step time (halo exchange included)
            peak, src = hooks["peaks"]()
            rvec = [0] + [1] * (ns - 1)
            e_rank = int(np.bincount(part, minlength=world).max())
            by = sum(e_rank * hooks["alg_bytes"](K, r) for r in rvec)
            ach = by / (t_ms / args.steps * 1e-3) / 1e9
            line["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                "frac": ach / peak, "traffic": None, "peak_source": src,
                                "kernel": "whole step per GPU (stage launches + halo exchange)",
                                "note": "ncu traffic and FP64 fraction: see the N=1 line"}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
