"""Diagnostic: device time of qf_rhs per term mask (volume / edge / source)
on a BASELINE config, to attribute the stage kernel's time to its phases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_08684_b200 import _cabi  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402


def timed(fn, reps, trials=7):
    """median over trials of the mean device time of `reps` back-to-back calls (us)."""
    out = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps * 1e3)
    out.sort()
    return out[len(out) // 2]


def main(cfg="c2", reps=40):
    lib = _cabi.load()
    k, n, mesh, scn = bench.build_problem(cfg)
    disc = Discretization(mesh, scn, k)
    st = disc.project_initial()
    ds = disc.to_device(st)
    out, _ = disc._empty_state()
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for name, terms in (("volume", 1), ("edge", 2), ("source", 4), ("all", 7), ("none", 0)):
        fn = lambda terms=terms: lib.qf_rhs(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), 0.1,  # noqa
                                            terms, out.data_ptr(), None, s)
        fn()
        res[name] = timed(fn, reps)
    w = disc._work_buf()
    st = lambda: lib.qf_stage(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), ds.c.data_ptr(),  # noqa
                              w.data_ptr(), w[3 * disc.K * disc.ld:].data_ptr(), 0.5, 0.5, 0.1,
                              disc.dt, None, 0.0, 0, -1, s)
    st()
    res["stage"] = timed(st, reps)
    print(cfg, {k_: round(v, 2) for k_, v in res.items()}, "us (qf_rhs includes a ghost launch when edge)")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c2"]))
