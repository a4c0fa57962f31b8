"""Diagnostic: stage-kernel device time per order k on a bump/wall problem
(no forcing) of N x N quads, median of trials; prints us/stage and DoF/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1904_08684_b200 import mesh as M, scenario as S  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402
from tools.term_timing import timed  # noqa: E402


def main(n=256, orders=(1, 2, 3, 4), scen="bumps", once=False):
    mesh = M.build_unit_square_mesh(n)
    for k in orders:
        scn = S.bump_scenario(seed=0, cfl=0.1) if scen == "bumps" else S.mms_scenario(dt=2e-5)
        disc = Discretization(mesh, scn, k)
        ds = disc.to_device(disc.project_initial())
        lib, s = disc._lib, torch.cuda.current_stream().cuda_stream
        w = disc._work_buf()
        st = lambda: lib.qf_stage(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), ds.c.data_ptr(),  # noqa
                                  w.data_ptr(), w[3 * disc.K * disc.ld:].data_ptr(), 0.5, 0.5,
                                  0.0, disc.dt, None, 0.0, 0, -1, s)
        st()
        if once:  # for ncu launch lists: one more stage, no timing loop
            st()
            torch.cuda.synchronize()
            continue
        us = timed(st, 20)
        dof = 3 * disc.K * mesh.n_triangles
        print(f"k={k} N={n} E={mesh.n_triangles} {scen}: {us:8.1f} us/stage  {dof / us * 1e6:.3e} DoF/s")


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("n", nargs="?", type=int, default=256)
    ap.add_argument("scen", nargs="?", default="bumps")
    ap.add_argument("--orders", default="1,2,3,4")
    ap.add_argument("--once", action="store_true")
    a = ap.parse_args()
    main(a.n, tuple(int(x) for x in a.orders.split(",")), a.scen, a.once)
