"""Benchmark: DG DoF-updates/s per RK stage on B200 (BASELINE.json metric).

Default workload = BASELINE configs[1] (C2): manufactured solution, p = 2,
2 x 256 x 256 = 131,072 triangles of the unit square, SSP-RK3, dt = 2e-5.
A "step" is one SSP-RK3 step = 3 stages; one DoF-update is one modal
coefficient of (xi, U, V) advanced through one stage (3*K*E per stage).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5]
    python bench.py --impl reference ...   # CPU oracle port on the host cores

Timing: CUDA events on the launching stream around each step, max over
ranks; the 131k-element C2 state (19 MB) fits in L2, so L2 is flushed
(a 256 MB write) between timed steps and the flush is outside the events.
Event-record nodes inside the replayed step graph time every RK stage (the
dominant kernel) for the roofline.  ``e2e`` is a dependent host-buffer
chain through the C ABI (each step uploads what the previous one
downloaded).  ``per_config`` repeats the measurement for the other BASELINE
orders (C1, C3, C4, C5) with the same method.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (order, n, scenario, dt or None (CFL), jitter, description)
    "c1": (1, 32, "mms", 1e-4, 0.0, "C1 MMS p=1 N=32 SSP-RK2 dt=1e-4"),
    "c2": (2, 256, "mms", 2e-5, 0.0, "C2 MMS p=2 N=256 SSP-RK3 dt=2e-5"),
    "c3": (3, 1024, "bumps", None, 0.0, "C3 bumps+walls p=3 N=1024 SSP-RK3 CFL 0.1"),
    "c4": (2, 2048, "bumps", None, 0.2, "C4 jittered bumps+walls p=2 N=2048 SSP-RK3 CFL 0.1"),
    "c5": (4, 1448, "bumps", None, 0.0, "C5 weak bumps+walls p=4 N=1448/GPU SSP-RK3 CFL 0.1"),
}
# Per RK stage (averaged over the stages of one L2-flushed step) of the stage
# launches (stage_kernel, + volume_kernel + velocity_kernel for k >= 3):
# DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and FP64 FLOP per
# element (2 dfma + dmul + dadd, smsp__sass_thread_inst_executed_op_*), from
# tools/kernel_counts.sh under ncu; summaries in profiles/r02_kernel_counts.txt
PROFILED = {
    "c1": {"bytes_per_elem": 284.6, "flop_per_elem": 2227.2},
    "c2": {"bytes_per_elem": 525.9, "flop_per_elem": 5173.3},
    "c3": {"bytes_per_elem": 1145.6, "flop_per_elem": 8332.9},
    "c4": {"bytes_per_elem": 723.3, "flop_per_elem": 3226.3},
    "c5": {"bytes_per_elem": 4126.4, "flop_per_elem": 18373.4},
}
# FP64 FMA-pipe peak of this B200, measured by tools/micro/fp64_pipes.cu
# (DFMA 35.3 TF/s, DMMA 37.1 TF/s, one shared pipe; profiles/r01_fp64_pipes.txt)
FP64_PEAK_TFLOPS = 35.3
METRIC = "DG DoF-updates/s per RK stage (p=1..4) at 1/2/4/8 B200; % of HBM roofline"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def stages_of(k):
    return 1 if k == 0 else (2 if k == 1 else 3)


def rk_coeffs(k):
    if k == 0:
        return [(0.0, 1.0, 0.0)]
    if k == 1:
        return [(0.0, 1.0, 0.0), (0.5, 0.5, 1.0)]
    return [(0.0, 1.0, 0.0), (0.75, 0.25, 1.0), (1.0 / 3.0, 2.0 / 3.0, 0.5)]


def alg_bytes_per_elem(K, r):
    """read c, write c_out, (+ read c0), + 64 B static + 12 B ids."""
    return 8 * 3 * K * (2 + r) + 64 + 12


def build_problem(cfg, n_override=None):
    from paper_1904_08684_b200 import mesh as M
    from paper_1904_08684_b200 import scenario as S

    k, n, scen, dt, jit, _ = CONFIGS[cfg]
    n = n_override or n
    mesh = M.build_unit_square_mesh(n, jitter=jit, seed=7 if jit else 0, lazy=True)
    if scen == "mms":
        scn = S.mms_scenario(dt=dt)
    else:
        scn = S.bump_scenario(seed=0, cfl=0.1)
    return k, n, mesh, scn


class Clocks:
    """SM clock + throttle reasons sampled through NVML during the timed
    region (the B200_PROFILING.md clocks line; nvidia-smi's 100 ms sampling
    is too coarse for a few-ms region, so one sample is taken per step)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, idx):
        self.samples, self.reasons, self.h = [], set(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def sample(self):
        if self.h is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def stop(self):
        if self.h is None or not self.samples:
            return None
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max),
                "samples": len(self.samples), "reasons": sorted(self.reasons), "source": "nvml"}


def cpu_baseline(cfg, budget_s=12.0, n_sample=64, max_steps=None, warm=1):
    """Oracle port (dense NumPy restatement of the reference) on this host."""
    from oracle import qfswe_oracle as O

    k, n, mesh, scn = build_problem(cfg, n_override=n_sample)
    if scn.name == "mms":
        oscn = O.mms_baseline(dt=scn.dt)
    else:
        oscn = O.OScenario(dt=1e-4, dirichlet_markers=frozenset(), wall_markers=frozenset({1}),
                           hb=scn.hb, initial=scn.initial)
    orc = O.OracleSolver(O.OMesh(mesh.vertices, mesh.triangles), oscn, k)
    c, _ = orc.project_initial()
    if scn.cfl is not None:
        _, u = orc.project_initial()
        orc.dt = orc.cfl_dt(scn.cfl, c, u)
    for _ in range(max(warm, 1)):
        orc.step(c, 0.0)  # warm-up
    t0 = time.perf_counter()
    steps, t = 0, 0.0
    while True:
        c, _, t = orc.step(c, t)
        steps += 1
        el = time.perf_counter() - t0
        if (max_steps and steps >= max_steps) or (not max_steps and el >= budget_s):
            break
    K = orc.K
    dof = 3 * K * mesh.n_triangles * stages_of(k) * steps
    try:
        from threadpoolctl import threadpool_info
        cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        cores = os.cpu_count()
    return {"value": dof / el, "unit": "DoF-updates/s", "cores": int(cores), "kind": "port",
            "sample": f"{CONFIGS[cfg][5]} restricted to N={n_sample} "
                      f"({mesh.n_triangles} elements), {steps} steps, wall clock, "
                      f"{os.cpu_count()} host cores visible", "elapsed_s": el}


def run_reference(args):
    """Reference arm: the CPU oracle port (dense NumPy restatement of the
    reference, all host threads) on this config, each step a bounded sample:
    the same workload on an N_s x N_s mesh with N_s chosen so the whole run
    stays near two minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    probe = cpu_baseline(args.config, n_sample=32, max_steps=1)
    per_elem_step = probe["elapsed_s"] / (2 * 32 * 32)
    budget = 120.0 / max(args.steps + args.warmup, 1)
    n_s = 32
    for cand in (96, 64, 48):
        if per_elem_step * 2 * cand * cand <= budget:
            n_s = cand
            break
    cbw = cpu_baseline(args.config, n_sample=n_s, max_steps=max(args.steps, 1),
                       warm=args.warmup)
    k, n, _, _ = build_problem(args.config)
    line = {
        "metric": METRIC, "value": cbw["value"], "unit": "DoF-updates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cbw["elapsed_s"] / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": CONFIGS[args.config][5], "order": k, "n": n,
                   "sample_n": n_s, "parallelism": "host cores (NumPy/OpenBLAS)"},
        "cpu_baseline": {k_: cbw[k_] for k_ in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cbw["value"], "unit": "DoF-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1904_08684_b200 import distributed as QD
        return QD.bench_distributed(args, CONFIGS, METRIC,
                                    hooks={"clocks": lambda: Clocks(local), "peaks": peaks,
                                           "alg_bytes": alg_bytes_per_elem})
    res = measure(args.config, args.steps, args.warmup, local, n=args.n, e2e=not args.no_e2e)
    line = {
        "metric": METRIC, "value": res["value"], "unit": "DoF-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
    }
    line.update({k_: v for k_, v in res.items() if k_ not in ("value", "ms_per_step")})
    if rank == 0 and not args.no_cpu:
        cb = cpu_baseline(args.config)
        line["cpu_baseline"] = {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
    if args.extra and args.n is None:
        # every other BASELINE order on the same box, same timing method
        # (graph-replayed steps, per-stage events inside the graph): the
        # metric is quoted for p = 1..4
        per = {}
        for cfg in sorted(CONFIGS):
            if cfg == args.config:
                continue
            try:
                r = measure(cfg, min(args.steps, 20), 3, local, e2e=False)
                per[cfg] = {k_: r[k_] for k_ in ("value", "ms_per_step", "roofline", "clocks",
                                                 "config", "checks", "gpu_launches", "setup_s",
                                                 "device_tables_s")}
            except Exception as err:  # keep the headline line even if one config fails
                per[cfg] = {"error": f"{type(err).__name__}: {err}"}
            torch.cuda.empty_cache()
        line["per_config"] = per
    print(json.dumps(line), flush=True)


def measure(cfg, steps, warmup, local, n=None, e2e=False):
    """One configuration on this GPU: ``steps`` timed SSP-RK steps, each one
    replay of the library's captured step graph (qf_run, as
    Discretization.run does) bracketed by CUDA events on the launching
    stream, L2 flushed (256 MB write) between steps outside the events.
    Event-record nodes inside the graph (qf_stage_events) time every RK stage
    of the same replays, which gives the dominant kernel's launch time for
    the roofline."""
    import torch

    from paper_1904_08684_b200 import _cabi
    from paper_1904_08684_b200.solver import Discretization

    lib = _cabi.load()
    t_setup = time.perf_counter()
    k, n_, mesh, scn = build_problem(cfg, n)
    disc = Discretization(mesh, scn, k)
    st0 = disc.project_initial()
    K, E, ld = disc.K, mesh.n_triangles, disc.ld
    ds = disc.to_device(st0)
    if st0._dev is not None:  # device-set-up state: step a copy, keep st0 initial
        ds = ds.clone()
    ds.t_dev[1] = disc.dt
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    work = disc._work_buf()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 256 MB > L2
    ns = stages_of(k)

    def step():  # 1 Dirichlet-data + ns stage launches + t advance, one graph replay
        _cabi.check(lib.qf_run(disc._ctx, 1, ds.c.data_ptr(), ds.u.data_ptr(), work.data_ptr(),
                               ds.t_dev.data_ptr(), 1, sp), "qf_run")

    def timed_steps(nsteps, sev=None, clocks=None):
        import gc

        step_ms, stage_ms = [], []
        # the step's events and graph launch are enqueued while the flush
        # kernels still run; no collector pause may fall into that window
        # (a host stall there would leave the GPU idle inside the events)
        gc.collect()
        gc.disable()
        try:
            return _timed_steps(nsteps, sev, clocks, step_ms, stage_ms)
        finally:
            gc.enable()

    def _timed_steps(nsteps, sev, clocks, step_ms, stage_ms):
        for it in range(nsteps):
            flush.fill_(float(it))  # outside the timed events
            flush.fill_(float(it) + 0.5)  # (twice: ~100 us of queue ahead of the step)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            step()
            ev1.record(stream)
            if clocks:
                clocks.sample()
            torch.cuda.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            if sev:
                stage_ms.append([sev[2 * i].elapsed_time(sev[2 * i + 1]) for i in range(ns)])
        return step_ms, stage_ms

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # pass A (the reported value): plain graph replays
    clocks = Clocks(local)
    n0 = lib.qf_launch_count()
    step_ms, _ = timed_steps(steps, clocks=clocks)
    launches = lib.qf_launch_count() - n0
    # pass B (roofline): the same step graph re-captured with event-record
    # nodes around every RK stage (qf_stage_events); kernel share = stage
    # time / step time of the same replays (the event nodes add a few us per
    # step, so pass B's step time is not the reported one)
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * ns)]
    for e_ in sev:
        e_.record(stream)  # creates the CUDA events
    handles = (_cabi.C.c_void_p * (2 * ns))(*[e_.cuda_event for e_ in sev])
    _cabi.check(lib.qf_stage_events(disc._ctx, handles, 2 * ns), "qf_stage_events")
    step()
    torch.cuda.synchronize()
    stepB_ms, stage_ms = timed_steps(min(steps, 50), sev=sev)
    _cabi.check(lib.qf_stage_events(disc._ctx, None, 0), "qf_stage_events")
    clk = clocks.stop()
    # diagnostic, not the headline: the same steps as a time-stepping run
    # issues them -- one qf_run call of `steps` graph replays back to back,
    # no L2 flush in between (the state of a small mesh stays in the 126 MB L2)
    nrun = max(steps, 20)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    _cabi.check(lib.qf_run(disc._ctx, nrun, ds.c.data_ptr(), ds.u.data_ptr(), work.data_ptr(),
                           ds.t_dev.data_ptr(), 1, sp), "qf_run")
    ev1.record(stream)
    torch.cuda.synchronize()
    run_ms = ev0.elapsed_time(ev1) / nrun
    disc._raise_errors("bench")
    checks = state_checks(disc, st0, ds, E)
    total_ms = float(np.sum(step_ms))
    value = 3 * K * E * ns * steps / (total_ms * 1e-3)
    peak, peak_src = peaks()
    st = np.array(stage_ms)
    rvec = [0] + [1] * (ns - 1)
    bytes_step = sum(E * alg_bytes_per_elem(K, r) for r in rvec)
    kern_ms_step = float(st.sum(axis=1).mean())
    achieved = bytes_step / (kern_ms_step * 1e-3) / 1e9
    prof = PROFILED.get(cfg) if n is None else None
    fp64 = None
    if prof:
        tf = prof["flop_per_elem"] * E * ns / (kern_ms_step * 1e-3) / 1e12
        fp64 = {"achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tf / FP64_PEAK_TFLOPS, "flop_per_elem_stage": prof["flop_per_elem"],
                "peak_source": "measured DFMA throughput (tools/micro/fp64_pipes.cu)"}
    out = {
        "value": value, "ms_per_step": total_ms / steps,
        "step_ms": {"min": float(np.min(step_ms)), "median": float(np.median(step_ms)),
                    "max": float(np.max(step_ms))},
        "config": {"workload": CONFIGS[cfg][5], "order": k, "n": n_, "elements": E,
                   "K": K, "stages_per_step": ns, "dt": disc.dt,
                   "dof_per_stage": 3 * K * E, "l2": "flushed (256 MB write) between timed steps",
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": prof["bytes_per_elem"] * E if prof else None,
                     "traffic_note": "DRAM bytes per stage launch (ncu, averaged over the "
                                     "stages of an L2-flushed step), algorithmic: "
                                     f"{bytes_step / ns:.4g}",
                     "peak_source": peak_src,
                     "kernel": "stage_kernel (one RK stage; timed by event-record nodes "
                               "inside the replayed step graph)",
                     "kernel_ms_per_step": kern_ms_step, "alg_bytes_per_step": bytes_step,
                     "kernel_share_of_step": kern_ms_step / float(np.mean(stepB_ms)),
                     "fp64": fp64},
        "hbm_roofline_dof_per_s": 3 * K * E * ns / (bytes_step / (peak * 1e9)),
        "gpu_launches": int(launches),
        "unflushed_run": {"value": 3 * K * E * ns / (run_ms * 1e-3), "ms_per_step": run_ms,
                          "steps": nrun, "note": "diagnostic: one qf_run call, no L2 flush "
                                                 "between its steps; not the reported value"},
        "checks": checks,
        "clocks": clk,
        "setup_s": setup_s,
        "device_tables_s": getattr(disc, "setup_seconds", None),
    }
    out["roofline_frac_dof"] = value / out["hbm_roofline_dof_per_s"]
    if e2e:
        out["e2e"] = measure_e2e(disc, st0, max(3, min(steps, 50)))
    del disc, ds, work, flush
    return out


def state_checks(disc, st0, ds, E):
    """Size-independent properties of the full-size run after the timed
    steps, evaluated on the device: xi mass conservation on
    wall configurations (total water volume sum_e sqrt(detB) c_xi,0 / sqrt 2),
    the L2 error against the exact solution (qf_l2_error) on manufactured ones."""
    import torch

    t_end = float(ds.t_dev[0].item())
    out = {"t": t_end, "steps_run": int(round(t_end / disc.dt))}
    g = disc._geo
    sd = torch.sqrt(g[0, :E] * g[3, :E] - g[1, :E] * g[2, :E])
    c0 = disc.to_device(st0).c
    if int(disc.tables.bnd_elem.shape[0]) == 0:
        m0 = float((c0[0, 0, :E] * sd).sum())
        m1 = float((ds.c[0, 0, :E] * sd).sum())
        out["xi_mass_drift_rel"] = abs(m1 - m0) / abs(m0)
    if getattr(disc.scn.device, "kind", 0) in (1, 2, 3) and disc.scn.exact is not None:
        out["l2_error_xi_U_V"] = [float(v) for v in np.sqrt(disc.l2_error_sq(ds, t_end))]
    return out


def measure_e2e(disc, st0, steps):
    """End to end through the C ABI with HOST buffers (pinned numpy arrays in
    the reference's (E, 3, K) State layout), as a DEPENDENT time-stepping
    chain: step i uploads the state that step i-1 downloaded.  Every step,
    in stream order: H2D of c, qf_pack, qf_velocity, qf_step (one SSP-RK step),
    qf_unpack, D2H of the new c into the buffer the next step uploads; CUDA
    events around all steps.  Nothing overlaps across steps (no step can start
    before its input has come back to the host).

    Also reported: ``public_api`` = ``Discretization.step`` on numpy States
    (the call a reference user makes; persistent pinned staging, c and u
    read back every step), and ``run_api`` = ``Discretization.run`` (one
    upload, graph-replayed steps, one download), both wall clock."""
    import torch

    from paper_1904_08684_b200 import _cabi
    from paper_1904_08684_b200.solver import State

    lib = disc._lib
    E, K, ld = disc.mesh.n_triangles, disc.K, disc.ld
    h = [torch.empty((E, 3, K), dtype=torch.float64).pin_memory() for _ in range(2)]
    h[0].numpy()[:] = st0.c
    d_in = torch.empty((E, 3, K), dtype=torch.float64, device="cuda")
    d_out = torch.empty((E, 3, K), dtype=torch.float64, device="cuda")
    c, u = disc._empty_state()
    c.zero_()
    u.zero_()
    tdev = torch.tensor([st0.t, disc.dt], dtype=torch.float64, device="cuda")
    work = disc._work_buf()
    pp = disc._perm_ptr(E)
    s_cmp = torch.cuda.current_stream()
    sp = s_cmp.cuda_stream

    def chain(n):
        for i in range(n):
            src, dst = h[i % 2], h[(i + 1) % 2]
            d_in.copy_(src, non_blocking=True)
            _cabi.check(lib.qf_pack(d_in.data_ptr(), c.data_ptr(), E, 3, K, ld, pp, sp), "pack")
            _cabi.check(lib.qf_velocity(disc._ctx, c.data_ptr(), u.data_ptr(), 0, -1, sp), "vel")
            _cabi.check(lib.qf_step(disc._ctx, c.data_ptr(), u.data_ptr(), work.data_ptr(),
                                    tdev.data_ptr(), sp), "step")
            _cabi.check(lib.qf_unpack(c.data_ptr(), d_out.data_ptr(), E, 3, K, ld, pp, sp),
                        "unpack")
            dst.copy_(d_out, non_blocking=True)

    chain(2)
    torch.cuda.synchronize()
    h[0].numpy()[:] = st0.c
    tdev[0] = st0.t
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    chain(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    disc._raise_errors("e2e")
    ns = stages_of(disc.k)
    dof = 3 * K * E * ns
    # the Python API (numpy State in, numpy State out), wall clock
    api_steps = min(steps, 20)
    st = disc.step(State(st0.c.copy(), st0.u.copy(), st0.t))
    _ = st.c
    t0 = time.perf_counter()
    for _ in range(api_steps):
        st = disc.step(State(st.c, st.u, st.t))
        _ = st.c
    api = time.perf_counter() - t0
    # Discretization.run(numpy State, t_end): one upload of c, graph-replayed
    # steps, the error word read once, one download of c and u, wall clock
    t_end = st0.t + steps * disc.dt
    _ = disc.run(State(st0.c.copy(), st0.u.copy(), st0.t), t_end=t_end).c
    t0 = time.perf_counter()
    _ = disc.run(State(st0.c.copy(), st0.u.copy(), st0.t), t_end=t_end).c
    run_s = time.perf_counter() - t0
    return {"value": dof * steps / (ms * 1e-3), "unit": "DoF-updates/s",
            "h2d_bytes_per_step": 8 * 3 * K * E, "d2h_bytes_per_step": 8 * 3 * K * E,
            "steps": steps,
            "timing": "C ABI, dependent chain: each step uploads (pinned H2D) the state the "
                      "previous step downloaded; H2D c, qf_pack, qf_velocity, qf_step, "
                      "qf_unpack, D2H c on one stream; CUDA events around all steps",
            "public_api": {"value": dof * api_steps / api, "unit": "DoF-updates/s",
                           "ms_per_step": 1e3 * api / api_steps,
                           "h2d_bytes_per_step": 8 * 3 * K * E,
                           "d2h_bytes_per_step": 8 * 5 * K * E,
                           "timing": "Discretization.step with numpy States (c and u read "
                                     "back every step), wall clock"},
            "run_api": {"value": dof * steps / run_s, "unit": "DoF-updates/s", "steps": steps,
                        "h2d_bytes_per_run": 8 * 3 * K * E, "d2h_bytes_per_run": 8 * 5 * K * E,
                        "timing": "Discretization.run(numpy State, t_end) over the steps: one "
                                  "upload of c, graph-replayed steps, error word read once, "
                                  "one download of c and u, wall clock"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--n", "--mesh-n", dest="n", type=int, default=None,
                    help="override mesh resolution (--mesh-n under torchrun, whose own "
                         "options would swallow --n)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the host-buffer legs (diagnostic runs at sizes whose host "
                         "State is tens of GB, e.g. C5 strong on one GPU)")
    ap.add_argument("--transport", default="p2p", choices=["nccl", "p2p"],
                    help="N > 1 halo exchange: the fused push (stage kernels store into the "
                         "peers' halo slots over CUDA IPC / NVLink; all ranks fall back to NCCL "
                         "together if a peer mapping fails), or NCCL send/recv")
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the per_config lines (the other BASELINE orders)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak (per-GPU mesh fixed, default) or strong (the BASELINE "
                         "global mesh: C3 N=1024, C5 N=4096, or --n)")
    ap.add_argument("--partition", default=None, choices=["strips", "blocks"],
                    help="N > 1 partition layout (default: blocks for c4, else strips)")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU runner even at world size 1 (smoke test)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
