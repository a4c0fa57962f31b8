"""Diagnostic: device time per graph-replayed step (qf_run) of the MMS problem
at several mesh sizes N -- the wave-quantisation probe of DESIGN §5 (blocks per
launch against the 3 x 148 resident block slots) -- or of any BASELINE config.

    python tools/step_timing.py 2 236 256 290 296      # order, N ...
    python tools/step_timing.py 2 256 --no-dataflow    # one launch per stage instead of step_kernel
    python tools/step_timing.py 3 512 --bumps          # bump / wall problem (no forcing)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1904_08684_b200 import mesh as M, scenario as S  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402
from tools.term_timing import timed  # noqa: E402


def main(k, sizes, steps=20, dataflow=True, scen="mms"):
    for n in sizes:
        mesh = M.build_unit_square_mesh(n)
        scn = S.mms_scenario(dt=2e-5) if scen == "mms" else S.bump_scenario(seed=0, cfl=0.1)
        disc = Discretization(mesh, scn, k)
        if hasattr(disc._lib, "qf_dataflow"):
            on = disc._lib.qf_dataflow(disc._ctx, 1 if dataflow else 0)
            print(f"[step kernel {'on' if on else 'off'}]", end=" ")
        ds = disc.to_device(disc.project_initial())
        ds.t_dev[1] = disc.dt
        disc.step_device(ds, 3)
        torch.cuda.synchronize()
        us = timed(lambda: disc.step_device(ds, steps), 1) / steps
        nst = 1 if k == 0 else (2 if k == 1 else 3)
        e = mesh.n_triangles
        print(f"k={k} N={n} E={e} blocks={-(-e // 128)} ({-(-e // 128) / 444:.2f} waves of 444): "
              f"{us:8.2f} us/step  {3 * disc.K * e * nst / us * 1e6:.3e} DoF/s", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(int(args[0]), [int(x) for x in args[1:]], dataflow="--no-dataflow" not in sys.argv,
         scen="bumps" if "--bumps" in sys.argv else "mms")
