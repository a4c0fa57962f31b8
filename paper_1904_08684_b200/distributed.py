"""Multi-GPU: contiguous element blocks with a cut-edge trace halo per stage.

The grid shards naturally: each rank owns a block of elements
(vertical strips of quad columns, or px x py rectangles on the unit-square
meshes).  A partition holds its owned elements only; what it needs from a
neighbour rank is, per cut edge and stage, the 6 (k + 1) trace moments (xi,
U, V, u, v, h_b) of the neighbour element on that edge, kept in a halo trace
table per RK buffer.  No per-stage collective exists: lambda is per edge
and dt is fixed; one allreduce(max) fixes a CFL dt and one allreduce(max)
takes the step time.

Overlap: owned elements are ordered interior-first; per stage the interior
range runs on the compute stream while the previous stage's halo is still in
flight, then the cut-adjacent range runs once the halo has arrived.  With
the p2p transport the cut-adjacent launch itself stores the new traces into
the peers' tables (CUDA IPC / NVLink) and the ranks order their stages with
stream memory operations on per-peer flags; the whole step of a rank --
launches, flag waits and writes, the two streams -- is captured once as a
CUDA graph and replayed with re-based flag values (``qf_graph_*``).  With
the NCCL transport ``qf_halo_traces`` computes the rows and
``batch_isend_irecv`` moves them on a communication stream.

The host logic (partitioning, halo lists, exchange) is shared by the GPU
runner and a CPU runner used by the ``gloo`` tests, whose stage executor is
the test-only oracle (``oracle/trace_stage.py``).
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
    """Local element order and halo-trace lists of one rank.

    A rank stores only its owned elements (interior first, then
    cut-adjacent).  For every cut edge (an edge whose other element belongs
    to another rank) it keeps one row of a halo trace table: the other
    element's trace moments of (xi, U, V, u, v, h_b) on that edge, 6 (k+1)
    doubles, refreshed every stage by the owner.  Rows are
    grouped by peer and, within a peer, ordered by global edge id, so both
    sides of a cut enumerate it the same way."""

    rank: int
    elements: np.ndarray          # owned global ids: interior, then cut-adjacent
    n_own: int
    n_int: int                    # owned elements without a remote neighbour
    send: dict = field(default_factory=dict)   # peer -> (n, 2) [local slot, local edge], peer-row order
    recv: dict = field(default_factory=dict)   # peer -> (first row, n rows) of my trace table
    ht_code: np.ndarray = None    # (3, n_own): my trace-table row per (local edge, slot), -1 = none

    @property
    def n_local(self) -> int:
        return len(self.elements)

    @property
    def n_ht(self) -> int:
        return sum(n for _, n in self.recv.values())

    def items(self, p) -> np.ndarray:
        """qf_halo_traces items (slot << 2 | local edge) of my send list to p."""
        sl = self.send[p]
        return (sl[:, 0] * 4 + sl[:, 1]).astype(np.int32)


def build_halo(mesh: Mesh, part: np.ndarray, rank: int) -> Halo:
    cn = mesh.conn
    nbr = cn.nbr
    own = np.flatnonzero(part == rank)
    nb = nbr[own]
    remote = (nb >= 0) & (part[np.maximum(nb, 0)] != rank)
    cut = remote.any(axis=1)
    from .mesh import locality_order

    oi, ob = own[~cut], own[cut]
    own_order = np.concatenate([oi[locality_order(mesh, oi)], ob[locality_order(mesh, ob)]])
    n_own, n_int = len(own), int((~cut).sum())
    g2l = np.full(mesh.n_triangles, -1, dtype=np.int64)
    g2l[own_order] = np.arange(n_own)
    # cut edges: (my global element, my local edge, peer, global edge id)
    e_loc, j_loc = np.nonzero(remote)
    ge = own[e_loc]
    peer = part[nbr[ge, j_loc]]
    eid = cn.elem_edge[ge, j_loc]
    order = np.lexsort((eid, peer))
    ge, j_loc, peer = ge[order], j_loc[order], peer[order]
    ht_code = np.full((3, n_own), -1, dtype=np.int64)
    send, recv = {}, {}
    row = 0
    for p in np.unique(peer):
        sel = peer == p
        n = int(sel.sum())
        slots = g2l[ge[sel]]
        # my rows for p's elements on these edges; the same edges, same order,
        # are p's send list to me
        ht_code[j_loc[sel], slots] = row + np.arange(n)
        recv[int(p)] = (row, n)
        send[int(p)] = np.column_stack([slots, j_loc[sel]]).astype(np.int64)
        row += n
    return Halo(rank=rank, elements=own_order, n_own=n_own, n_int=n_int, send=send, recv=recv,
                ht_code=ht_code)


PUSH_SLOT_BITS = 26


def push_table(halo: Halo, peer_recv: dict, ld: int) -> np.ndarray:
    """Destinations of the fused halo push (``qf_stage_push``): int32 [3][ld],
    entry (peer << 26) | row of the peer's halo trace table for (local edge,
    element), -1 = none.  ``peer_recv[p]`` is peer p's ``halo.recv[my rank]``
    (first row, count); my ``send[p]`` lists the same cut edges in the same
    order."""
    tab = np.full((3, ld), -1, dtype=np.int32)
    for p, sl in halo.send.items():
        first, n = peer_recv[p]
        if n != len(sl):
            raise ValueError(f"halo lists of rank {halo.rank} and peer {p} disagree")
        if p >= 1 << (31 - PUSH_SLOT_BITS) or first + n > 1 << PUSH_SLOT_BITS:
            raise ValueError("push table overflow (peer or row index)")
        if (tab[sl[:, 1], sl[:, 0]] != -1).any():
            raise ValueError("a cut edge has two peers")
        tab[sl[:, 1], sl[:, 0]] = (p << PUSH_SLOT_BITS) | (first + np.arange(n))
    return tab


def peer_table(torch, entries, device):
    """Device qf_peer[] table: entries[p] = halo trace table pointer of peer p, or None."""
    t = torch.zeros((max(len(entries), 1), 1), dtype=torch.int64)
    for p, ent in enumerate(entries):
        if ent is not None:
            t[p, 0] = int(ent)
    return t.to(device)


# ----------------------------------------------------------------- exchange
class HaloExchange:
    """Halo trace rows of the send lists -> P2P exchange -> row ranges of the
    peers' halo trace tables.

    On the GPU the rows are computed by ``qf_halo_traces`` (the stage
    kernel's rounding) and moved by ``torch.distributed.batch_isend_irecv``
    (NCCL P2P over NVLink) straight into the receiving table; on the CPU
    (``gloo`` tests) ``tracer(c, u, items) -> (n, 6, NT)`` computes them.
    """

    def __init__(self, halo: Halo, NT: int, device, lib=None, ctx=None, tracer=None):
        import torch

        self.torch = torch
        self.halo, self.W, self.lib, self.ctx, self.tracer = halo, 6 * NT, lib, ctx, tracer
        self.dev = device
        self.peers = sorted(set(halo.send) | set(halo.recv))
        self.items = {p: torch.as_tensor(halo.items(p), device=device) for p in halo.send}
        self.sbuf = {p: torch.empty(len(self.items[p]) * self.W, dtype=torch.float64,
                                    device=device) for p in halo.send}

    def traces(self, c, u, p, stream=None):
        """My rows for peer p (its trace-table rows for our cut edges)."""
        n = len(self.items[p])
        buf = self.sbuf[p]
        if self.lib is not None:
            s = stream.cuda_stream if stream is not None else \
                self.torch.cuda.current_stream().cuda_stream
            from . import _cabi
            _cabi.check(self.lib.qf_halo_traces(self.ctx, c.data_ptr(), u.data_ptr(),
                                                self.items[p].data_ptr(), n, buf.data_ptr(), s),
                        "qf_halo_traces")
        elif n:
            npy = lambda a: a.numpy() if hasattr(a, "numpy") else a  # noqa: E731
            rows = self.tracer(npy(c), npy(u), self.items[p].numpy())
            buf.copy_(self.torch.as_tensor(np.ascontiguousarray(rows)).reshape(-1))
        return buf

    def exchange(self, c, u, ht, stream=None):
        """Blocking (w.r.t. ``stream``) refresh of the halo trace table ``ht``
        ((n_ht, 6 NT) tensor) from the peers' (c, u)."""
        import torch.distributed as dist

        for p in self.halo.send:
            self.traces(c, u, p, stream)
        ops = []
        flat = ht.view(-1)
        for p in self.peers:
            if p in self.sbuf and len(self.sbuf[p]):
                ops.append(dist.P2POp(dist.isend, self.sbuf[p], p))
            if p in self.halo.recv and self.halo.recv[p][1]:
                first, n = self.halo.recv[p]
                ops.append(dist.P2POp(dist.irecv, flat[first * self.W:(first + n) * self.W], p))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


def rk_plan(k: int):
    """(src, dst, a, b, toff) per stage over buffers 0 (state), 1, 2."""
    if k == 0:
        return [(0, 1, 0.0, 1.0, 0.0)]
    if k == 1:
        return [(0, 1, 0.0, 1.0, 0.0), (1, 0, 0.5, 0.5, 1.0)]
    return [(0, 1, 0.0, 1.0, 0.0), (1, 2, 0.75, 0.25, 1.0), (2, 0, 1.0 / 3.0, 2.0 / 3.0, 0.5)]


# ------------------------------------------------------------- GPU runner
class PartitionRunner:
    """Device state, halo trace tables and stage launches of one partition."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray, rank: int):
        import torch

        from .solver import Discretization

        self.torch = torch
        self.k = order
        self.halo = build_halo(mesh, part, rank)
        h = self.halo
        self.disc = Discretization(mesh, scenario, order, elements=h.elements, n_own=h.n_own,
                                   halo_code=h.ht_code)
        d = self.disc
        self.K, self.ld, self.lib = d.K, d.ld, d._lib
        self.NT = order + 1
        self.c = d._c_init.clone() if d.device_setup else d.upload_fields(d.project_fields())
        self.u = torch.zeros_like(self.c[:2])
        self.bufs = {0: (self.c, self.u),
                     1: (torch.zeros_like(self.c), torch.zeros_like(self.u)),
                     2: (torch.zeros_like(self.c), torch.zeros_like(self.u))}
        # halo trace table per RK buffer: rows for the stage reading that buffer
        self.ht = {b: torch.zeros((max(h.n_ht, 1), 6 * self.NT), dtype=torch.float64,
                                  device=d.device) for b in range(3)}
        s = torch.cuda.current_stream().cuda_stream
        d._check(self.lib.qf_velocity(d._ctx, self.c.data_ptr(), self.u.data_ptr(), 0,
                                      h.n_own, s), "qf_velocity")
        self.dt = d.dt
        self.t = 0.0
        self.t_dev = None  # device {t, dt}: set by use_device_time (graph-replayable steps)

    def use_device_time(self):
        """Stage and Dirichlet-data times from a device {t, dt} pair advanced on
        the stream (as the single-domain qf_step does) instead of host
        scalars baked into every launch: a captured step can be replayed."""
        self.t_dev = self.torch.tensor([self.t, self.dt], dtype=self.torch.float64,
                                       device=self.disc.device)

    def traces_for(self, p, b=0, out=None):
        """My halo trace rows for peer p from RK buffer b (device tensor)."""
        torch, h = self.torch, self.halo
        items = torch.as_tensor(h.items(p), device=self.disc.device)
        n = len(items)
        out = torch.empty((max(n, 1), 6 * self.NT), dtype=torch.float64,
                          device=self.disc.device) if out is None else out
        c, u = self.bufs[b]
        self.disc._check(self.lib.qf_halo_traces(self.disc._ctx, c.data_ptr(), u.data_ptr(),
                                                 items.data_ptr(), n, out.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream),
                         "qf_halo_traces")
        return out[:n]

    def local_lambda_max(self) -> float:
        d, torch = self.disc, self.torch
        lam = torch.zeros((3, self.ld), dtype=torch.float64, device=d.device)
        out = torch.empty_like(self.c)
        d._check(self.lib.qf_halo_table(d._ctx, self.ht[0].data_ptr()), "qf_halo_table")
        d._check(self.lib.qf_rhs(d._ctx, self.c.data_ptr(), self.u.data_ptr(), 0.0, 2,
                                 out.data_ptr(), lam.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream), "qf_rhs")
        return float(lam[:, : self.halo.n_own].max().item())

    def ghost(self, si: int, stream):
        """Dirichlet data of stage ``si`` (read by both ranges of the stage)."""
        d = self.disc
        if int(d.tables.bnd_elem.shape[0]):
            toff = rk_plan(self.k)[si][4]
            if self.t_dev is not None:
                d._check(self.lib.qf_ghost_dev(d._ctx, self.t_dev.data_ptr(), toff,
                                               stream.cuda_stream), "qf_ghost_dev")
            else:
                self.lib.qf_ghost(d._ctx, self.t + toff * self.dt, stream.cuda_stream)

    def stage(self, si: int, part: str, stream, ghost: bool = True, push=None, peers=None):
        """Launch stage ``si`` on the 'interior', 'boundary' or 'all' owned range
        (with ``ghost``, the interior / all launch is preceded by the stage's
        Dirichlet data).  Halo neighbours are read from the trace table of the
        stage input; ``push``/``peers`` (device tensors): fused push of the
        new cut-edge traces into the peers' tables for the stage output."""
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
        if n > 0:
            td = None if self.t_dev is None else self.t_dev.data_ptr()
            d._check(lib.qf_stage_push(d._ctx, ci.data_ptr(), ui.data_ptr(), self.c.data_ptr(),
                                       co.data_ptr(), uo.data_ptr(), a, b, ts, self.dt, td,
                                       toff if td else 0.0, e0, n, self.ht[src].data_ptr(),
                                       None if push is None else push.data_ptr(),
                                       None if peers is None else peers.data_ptr(), s),
                     "qf_stage_push")
        return co, uo

    def end_step(self):
        if self.k == 0:
            self.torch.cuda.current_stream().wait_stream(getattr(self, "comm", None)
                                                         or self.torch.cuda.current_stream())
            self.c.copy_(self.bufs[1][0])
            self.u.copy_(self.bufs[1][1])
            self.ht[0].copy_(self.ht[1])
        if self.t_dev is not None:
            self.disc._check(self.lib.qf_advance_time(
                self.t_dev.data_ptr(), self.torch.cuda.current_stream().cuda_stream),
                "qf_advance_time")
        self.t += self.dt


class DistributedRunner(PartitionRunner):
    """One rank of a partitioned run (one process per GPU, NCCL P2P halos)."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray, rank: int,
                 world: int, transport: str = "nccl", graph: bool = True):
        import torch
        import torch.distributed as dist

        super().__init__(mesh, scenario, order, part, rank)
        self.dist, self.rank, self.world = dist, rank, world
        self.use_graph = graph  # p2p transport: replay the rank's step as one CUDA graph
        self._graph = None
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
            # initial halo traces (state of buffer 0); repeated after every stage
            self.ex = HaloExchange(self.halo, self.NT, self.disc.device, lib=self.lib,
                                   ctx=self.disc._ctx)
            self.ex.exchange(self.c, self.u, self.ht[0])
            torch.cuda.synchronize()
        else:
            self._initial_push()
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
        """Fused transport: map the peers' halo trace tables (CUDA IPC over
        NVLink) and build the push table; per stage the cut-adjacent launch
        stores its new cut-edge traces straight into the peers' tables and raises a
        per-peer flag (stream memory operation); the peer's next cut-adjacent
        launch waits on that flag (no NCCL, no gather / scatter kernels).
        Collective-safe: every rank reaches the same collectives and all
        ranks agree on the outcome (False: use NCCL)."""
        import ctypes as C

        torch, dist, lib = self.torch, self.dist, self.lib
        h = self.halo
        self.peers = sorted(set(h.send) | set(h.recv))
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=self.disc.device)
        bufs = [self.ht[b] for b in range(3)] + [self.flags]
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
        dist.all_gather_object(info, {"ipc": mine, "recv": {int(p): list(v)
                                                            for p, v in h.recv.items()}})
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
            self.peer_ht = ptrs
            self.peer_recv = {p: info[p]["recv"][self.rank] for p in h.send}
            self.peer_bufs = [peer_table(torch, [ptrs[p][b] if p in ptrs else None
                                                 for p in range(self.world)], dev)
                              for b in range(3)]
            # my flag slot in each peer's flag array; handshake write of 0
            self.remote_flag = {p: ptrs[p][3] + 4 * self.rank for p in self.peers}
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

    def _initial_push(self):
        """Initial halo traces over the mapped peer tables: my rows for each
        peer copied into its table 0, then a barrier (no rank steps before
        every table holds the initial state's traces)."""
        torch, lib = self.torch, self.lib
        W = 6 * self.NT
        s = torch.cuda.current_stream().cuda_stream
        for p in self.halo.send:
            rows = self.traces_for(p, 0)
            first, n = self.peer_recv[p]
            if n:
                self.disc._check(lib.qf_copy(self.peer_ht[p][0] + 8 * first * W, rows.data_ptr(),
                                             8 * n * W, s), "qf_copy")
        torch.cuda.synchronize()
        self.dist.barrier()

    def _step_p2p(self):
        """One step over the fused transport.  With ``graph`` the enqueue
        below is captured once (stage launches, flag waits / writes, both
        streams) and every later step is one qf_graph_launch with the flag
        values re-based by the stages completed since the capture."""
        import ctypes as C

        torch, lib = self.torch, self.lib
        if not self.use_graph:
            return self._enqueue_p2p(torch.cuda.current_stream())
        if self._graph is None:
            # (the legacy default stream cannot capture: the graph lives on its own stream)
            self.gstream = torch.cuda.Stream()
            if self.t_dev is None:
                self.use_device_time()
            torch.cuda.synchronize()
            gen0, t0 = self.gen, self.t
            h, err = C.c_void_p(), None
            with torch.cuda.stream(self.gstream):
                self.disc._check(lib.qf_graph_begin(self.gstream.cuda_stream), "qf_graph_begin")
                try:
                    self._enqueue_p2p(self.gstream)
                except Exception as exc:  # noqa: BLE001 (the capture must still be ended)
                    err = exc
                st = lib.qf_graph_end(self.gstream.cuda_stream, C.byref(h))
            self.gen, self.t = gen0, t0  # the capture enqueued nothing: run the step now
            if err is not None or st != 0 or not h.value:
                # (e.g. a driver that cannot capture stream memory operations)
                self.use_graph = False
                self.graph_note = f"step graph unavailable: {err or lib.qf_last_error().decode()}"
                return self._enqueue_p2p(torch.cuda.current_stream())
            self._graph, self._graph_gen0 = h, gen0
        self.gstream.wait_stream(torch.cuda.current_stream())
        self.disc._check(lib.qf_graph_launch(self._graph, self.gen - self._graph_gen0,
                                             self.gstream.cuda_stream), "qf_graph_launch")
        self.gen += len(rk_plan(self.k))
        self.t += self.dt

    def _enqueue_p2p(self, main):
        torch, lib = self.torch, self.lib
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
                self.ex.exchange(co, uo, self.ht[rk_plan(self.k)[si][1]], self.comm)
            main.wait_stream(self.bnd)               # next stage's interior reads these rows
        self.end_step()

    def sync(self):
        main = self.torch.cuda.current_stream()
        if self.transport == "nccl":
            main.wait_stream(self.comm)
        main.wait_stream(self.bnd)
        if getattr(self, "gstream", None) is not None:
            main.wait_stream(self.gstream)


class LocalMultiRunner:
    """All partitions in one process on one GPU (single-GPU tests of the
    partitioned kernels): the halo trace rows are either
    pushed by the stage kernels into each other's tables (``push``, the
    fused transport) or computed by ``qf_halo_traces`` from the peer's
    stage output and copied (``gather``, what the NCCL transport moves)."""

    def __init__(self, mesh: Mesh, scenario, order: int, part: np.ndarray,
                 transport: str = "gather"):
        import torch

        self.torch = torch
        world = int(part.max()) + 1
        self.parts = [PartitionRunner(mesh, scenario, order, part, r) for r in range(world)]
        self.k = order
        self.transport = transport
        if transport == "push":
            for r, pr in enumerate(self.parts):
                recv = {p: self.parts[p].halo.recv[r] for p in pr.halo.send}
                pr.push_tab = torch.as_tensor(push_table(pr.halo, recv, pr.ld), device="cuda")
                pr.peer_bufs = [peer_table(torch, [q.ht[b].data_ptr() for q in self.parts], "cuda")
                                for b in range(3)]
        self._refresh(0)  # halo traces of the initial state

    def _refresh(self, b):
        """Every partition's table b from its peers' buffer b."""
        for r, pr in enumerate(self.parts):
            for p, (first, n) in pr.halo.recv.items():
                if n:
                    pr.ht[b][first:first + n].copy_(self.parts[p].traces_for(r, b))

    def step(self):
        s = self.torch.cuda.current_stream()
        for si in range(len(rk_plan(self.k))):
            dst = rk_plan(self.k)[si][1]
            for pr in self.parts:
                if self.transport == "push":
                    pr.stage(si, "all", s, push=pr.push_tab, peers=pr.peer_bufs[dst])
                else:
                    pr.stage(si, "all", s)
            if self.transport != "push":
                self._refresh(dst)
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
    # watchdog on the first steps: a halo flag that never arrives (a peer
    # mapping that silently does not work on some topology) must end the
    # run with a message, not hang the node until the driver's limit
    done = torch.cuda.Event()
    done.record()
    t_wait = time.perf_counter()
    while not done.query():
        if time.perf_counter() - t_wait > float(os.environ.get("QF_DIST_WATCHDOG_S", "180")):
            import sys
            print(f"rank {rank}: warm-up steps did not complete within the watchdog time "
                  f"(transport {run.transport}, step graph {run._graph is not None}); "
                  "try --transport nccl", file=sys.stderr, flush=True)
            os._exit(3)
        time.sleep(0.01)
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
                           "step_graph": run._graph is not None,
                           "step_graph_note": getattr(run, "graph_note", None),
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
