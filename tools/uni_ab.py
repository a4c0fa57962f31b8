"""Diagnostic: C2 step time with the tabulated MMS phase offsets (qf_desc.uni)
against the degree-7 Taylor offsets, same mesh / state; also the max
relative difference of the two results after the timed steps (roundoff)."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1904_08684_b200 import mesh as M, scenario as S  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402
from tools.term_timing import timed  # noqa: E402


def main(n=256, k=2, steps=10):
    mesh = M.build_unit_square_mesh(n)
    scn = S.mms_scenario(dt=2e-5)
    outs = {}
    for name in ("taylor", "table", "taylor", "table"):
        if name == "taylor":
            orig = Discretization._uniform_phase_table
            Discretization._uniform_phase_table = lambda self: None
            disc = Discretization(mesh, scn, k)
            Discretization._uniform_phase_table = orig
        else:
            disc = Discretization(mesh, scn, k)
        assert (disc._desc.uni is not None) == (name == "table")
        ds0 = disc.to_device(disc.project_initial())
        ds0.t_dev[1] = disc.dt
        ds = ds0.clone()
        disc.step_device(ds, 2)
        torch.cuda.synchronize()
        us = timed(lambda: disc.step_device(ds, steps), 1) / steps
        print(f"{name:7s} k={k} N={n}: {us:8.2f} us/step  {us / 3:7.2f} us/stage")
        ds = ds0.clone()
        disc.step_device(ds, 50)
        outs[name] = ds.c.cpu().numpy()
    a, b = outs["taylor"], outs["table"]
    print("max rel diff after 50 steps:", float(np.abs(a - b).max() / np.abs(a).max()))


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
