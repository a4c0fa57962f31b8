"""Diagnostic: device time of qf_rhs per term mask (volume / edge / source)
on a BASELINE config, to attribute the stage kernel's time to its phases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_08684_b200 import _cabi  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402


def main(cfg="c2", reps=50):
    lib = _cabi.load()
    k, n, mesh, scn = bench.build_problem(cfg)
    disc = Discretization(mesh, scn, k)
    st = disc.project_initial()
    ds = disc.to_device(st)
    out, _ = disc._empty_state()
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for name, terms in (("volume", 1), ("edge", 2), ("source", 4), ("all", 7), ("none", 0)):
        for _ in range(3):
            lib.qf_rhs(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), 0.1, terms, out.data_ptr(), None, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            lib.qf_rhs(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), 0.1, terms, out.data_ptr(), None, s)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps * 1e3
    # full stage (RK + velocity epilogue)
    w = disc._work_buf()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.qf_stage(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), ds.c.data_ptr(), w.data_ptr(),
                     w[3 * disc.K * disc.ld:].data_ptr(), 0.5, 0.5, 0.1, disc.dt, None, 0.0, 0, -1, s)
    e1.record()
    torch.cuda.synchronize()
    res["stage"] = e0.elapsed_time(e1) / reps * 1e3
    print(cfg, {k_: round(v, 2) for k_, v in res.items()}, "us (qf_rhs includes a ghost launch when edge)")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c2"]))
