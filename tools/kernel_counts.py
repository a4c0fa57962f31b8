"""Diagnostic for ncu: one L2-flushed SSP-RK step of a bench config inside an
NVTX range "measure", so that

  ncu --nvtx --nvtx-include "measure/" --metrics <fp64 op counts, dram bytes> \\
      --csv --log-file out.csv python tools/kernel_counts.py c3

lists exactly the kernels of one step; ``--parse out.csv`` then prints FP64
FLOP and DRAM bytes per element per stage for each kernel."""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

METRICS = ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,"
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,"
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,"
           "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum")


def run(cfg, n=None):
    import torch

    import bench
    from paper_1904_08684_b200.solver import Discretization

    k, n, mesh, scn = bench.build_problem(cfg, n)
    disc = Discretization(mesh, scn, k)
    ds = disc.to_device(disc.project_initial())
    ds.t_dev[1] = disc.dt
    work = disc._work_buf()
    sp = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    step = lambda: disc._lib.qf_step(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(),  # noqa: E731
                                     work.data_ptr(), ds.t_dev.data_ptr(), sp)
    step()
    flush.fill_(1.0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("measure")
    step()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    print(f"{cfg}: k={k} n={n} E={mesh.n_triangles}")


def parse(path, E, stages):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    per = defaultdict(lambda: defaultdict(float))
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "usecond": 1.0,
                 "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        per[name][r["Metric Name"]] += v * scale
    tot = defaultdict(float)
    for name, m in per.items():
        fl = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
              + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
              + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"])
        by = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        us = m["gpu__time_duration.sum"]
        for key, v in (("flop", fl), ("bytes", by), ("us", us)):
            tot[key] += v
        print(f"{name:28s} FP64 FLOP/elem/stage {fl / E / stages:9.1f}  DRAM B/elem/stage "
              f"{by / E / stages:8.1f}  us/step {us:9.1f}")
    print(f"{'step total':28s} FP64 FLOP/elem/stage {tot['flop'] / E / stages:9.1f}  DRAM B/elem/stage "
          f"{tot['bytes'] / E / stages:8.1f}  us/step {tot['us']:9.1f}")


if __name__ == "__main__":
    if sys.argv[1] == "--parse":
        parse(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        run(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
