"""CPU, world_size 2 (gloo): partition + halo exchange host logic of
``distributed.py`` driving the test-only trace-space oracle as the stage
executor.  A partitioned run must reproduce the single-domain run exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import trace_stage as TS
from paper_1904_08684_b200 import distributed as D
from paper_1904_08684_b200 import mesh as M
from paper_1904_08684_b200 import scenario as S
from paper_1904_08684_b200.solver import HostSetup


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenario(case):
    if case == "mms":
        return S.mms_scenario(dt=1e-4)
    return S.bump_scenario(seed=0, dt=2e-4, cfl=None)


def _run_partitioned(rank, world, n, k, case, steps, part_kind):
    mesh = M.build_unit_square_mesh(n)
    scn = _scenario(case)
    part = {"strips": D.strip_partition(n, world), "blocks": D.block_partition(n, 2, world // 2),
            "ranges": D.range_partition(mesh.n_triangles, world)}[part_kind]
    halo = D.build_halo(mesh, part, rank)
    hs = HostSetup(mesh, scn, k, elements=halo.elements, n_own=halo.n_own,
                   halo_code=halo.ht_code)
    tb = hs.tables
    ts = TS.TraceStage(k, tb.geo, tb.nbr, hs.hb_table(), halo.n_own, scn, tb.bnd_elem,
                       tb.bnd_local)
    K, ld, nl, NT = hs.K, tb.ld, halo.n_local, k + 1
    c = np.zeros((3, K, ld))
    c[:, :, :nl] = hs.project_fields().transpose(1, 2, 0)
    u = np.zeros((2, K, ld))
    u[:, :, :nl] = ts.velocity(c, np.arange(nl))
    bufs = {0: (c, u), 1: (np.zeros_like(c), np.zeros_like(u)),
            2: (np.zeros_like(c), np.zeros_like(u))}
    ht = {b: torch.zeros((max(halo.n_ht, 1), 6 * NT), dtype=torch.float64) for b in range(3)}
    ex = D.HaloExchange(halo, NT, "cpu", tracer=ts.halo_traces) if world > 1 else None
    if ex is not None:
        ex.exchange(c, u, ht[0])
    t, dt = 0.0, scn.dt
    for _ in range(steps):
        for src, dst, a, b, toff in D.rk_plan(k):
            ci, ui = bufs[src]
            co, uo = bufs[dst]
            ts.ht = ht[src].numpy().reshape(-1, 6, NT)
            cn, un = ts.stage_coeffs(a, b, ci, ui, c, t + toff * dt, dt)
            co[:, :, : halo.n_own] = cn
            uo[:, :, : halo.n_own] = un
            if ex is not None:
                ex.exchange(co, uo, ht[dst])
        t += dt
    own = halo.elements[: halo.n_own]
    return own, c[:, :, : halo.n_own].copy(), u[:, :, : halo.n_own].copy()


def _worker(rank, world, port, args, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    own, c, u = _run_partitioned(rank, world, *args)
    res = [None] * world
    dist.all_gather_object(res, (own, c, u))
    if rank == 0:
        out.put(res)
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("k,case,part", [(1, "mms", "strips"), (2, "walls", "strips"),
                                         (2, "mms", "ranges"), (1, "walls", "blocks")])
def test_partitioned_equals_single_domain(k, case, part):
    n, steps = 8, 3
    own1, c1, u1 = _run_partitioned(0, 1, n, k, case, steps, "ranges")
    ref_c = np.zeros((3, c1.shape[1], 2 * n * n))
    ref_c[:, :, own1] = c1
    res = _spawn(2, (n, k, case, steps, part))
    got = np.zeros_like(ref_c)
    seen = np.zeros(2 * n * n, bool)
    for own, c, _u in res:
        got[:, :, own] = c
        assert not seen[own].any()
        seen[own] = True
    assert seen.all()
    assert np.array_equal(got, ref_c)


def _row_edges(mesh, h):
    """Global edge id of each row of rank h's halo trace table."""
    cn = mesh.conn
    out = np.full(h.n_ht, -1, dtype=np.int64)
    j, e = np.nonzero(h.ht_code >= 0)
    out[h.ht_code[j, e]] = cn.elem_edge[h.elements[e], j]
    return out


def test_halo_lists_are_symmetric():
    n, world = 12, 4
    mesh = M.build_unit_square_mesh(n)
    cn = mesh.conn
    for part in (D.strip_partition(n, world), D.block_partition(n, 2, 2),
                 D.range_partition(mesh.n_triangles, world)):
        halos = [D.build_halo(mesh, part, r) for r in range(world)]
        for h in halos:
            assert (part[h.elements] == h.rank).all() and h.n_local == h.n_own
            # interior-first ordering: no interior element touches another rank
            nb = cn.nbr[h.elements[: h.n_int]]
            assert ((nb < 0) | (part[np.maximum(nb, 0)] == h.rank)).all()
            # every remote neighbour of an owned element has exactly one row
            nb = cn.nbr[h.elements]
            remote = (nb >= 0) & (part[np.maximum(nb, 0)] != h.rank)
            assert np.array_equal(h.ht_code.T >= 0, remote)
            rows = _row_edges(mesh, h)
            assert (rows >= 0).all() and len(np.unique(rows)) == h.n_ht
            for p, (first, cnt) in h.recv.items():
                peer = halos[p]
                sl = peer.send[h.rank]
                sent = cn.elem_edge[peer.elements[sl[:, 0]], sl[:, 1]]
                assert np.array_equal(rows[first:first + cnt], sent)


@pytest.mark.parametrize("part", ["strips", "blocks", "ranges"])
def test_push_tables_fill_every_halo_row_once(part):
    """Fused halo push (qf_stage_push) tables: emulating the kernel's stores
    (every owned element and cut edge -> its (peer, row) entry) fills each
    rank's halo trace table exactly once, each row with the edge it stands for."""
    n = 12
    mesh = M.build_unit_square_mesh(n)
    cn = mesh.conn
    p = {"strips": D.strip_partition(n, 3), "blocks": D.block_partition(n, 2, 2),
         "ranges": D.range_partition(mesh.n_triangles, 3)}[part]
    world = int(p.max()) + 1
    halos = [D.build_halo(mesh, p, r) for r in range(world)]
    got = [np.full(h.n_ht, -1, dtype=np.int64) for h in halos]
    hits = [np.zeros(h.n_ht, dtype=np.int64) for h in halos]
    for r, h in enumerate(halos):
        ld = (h.n_local + 31) // 32 * 32
        tab = D.push_table(h, {q: halos[q].recv[r] for q in h.send}, ld)
        assert tab.shape == (3, ld) and (tab[:, h.n_own:] == -1).all()
        assert (tab[:, : h.n_int] == -1).all()  # interior elements push nothing
        for j in range(3):
            for e in np.flatnonzero(tab[j] >= 0):
                q, row = tab[j, e] >> D.PUSH_SLOT_BITS, tab[j, e] & ((1 << D.PUSH_SLOT_BITS) - 1)
                got[q][row] = cn.elem_edge[h.elements[e], j]
                hits[q][row] += 1
    for h, g, c in zip(halos, got, hits):
        assert (c == 1).all()
        assert np.array_equal(g, _row_edges(mesh, h))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_host_setup_partition_independent(k):
    """Host projections (P1 bathymetry, initial state) of a partition equal
    the whole-mesh ones bit for bit (fixed per-row summation order)."""
    n = 16
    mesh = M.build_unit_square_mesh(n)
    for scn in (S.bump_scenario(seed=0, dt=2e-4, cfl=None), S.mms_scenario(dt=1e-4)):
        full = HostSetup(mesh, scn, k)
        fc = full.project_fields()
        for p in (D.block_partition(n, 2, 2), D.range_partition(mesh.n_triangles, 5)):
            for r in range(int(p.max()) + 1):
                h = D.build_halo(mesh, p, r)
                hs = HostSetup(mesh, scn, k, elements=h.elements, n_own=h.n_own,
                               halo_code=h.ht_code)
                assert np.array_equal(hs.hb_coef, full.hb_coef[h.elements])
                assert np.array_equal(hs.project_fields(), fc[h.elements])
