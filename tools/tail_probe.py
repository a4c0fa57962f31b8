"""Diagnostic: wave quantisation of the stage kernel.  Per-element device
time of one C2-type stage (MMS, p = 2) against N: 2 N^2 / 128 blocks over
148 SMs x 3 resident blocks; a sawtooth in us per element shows the tail."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1904_08684_b200 import mesh as M, scenario as S  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402
from tools.term_timing import timed  # noqa: E402


def main(ns, k=2):
    for n in ns:
        mesh = M.build_unit_square_mesh(n)
        disc = Discretization(mesh, S.mms_scenario(dt=2e-5), k)
        ds = disc.to_device(disc.project_initial())
        lib, s = disc._lib, torch.cuda.current_stream().cuda_stream
        w = disc._work_buf()
        st = lambda: lib.qf_stage(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), ds.c.data_ptr(),  # noqa
                                  w.data_ptr(), w[3 * disc.K * disc.ld:].data_ptr(), 0.5, 0.5,
                                  0.0, disc.dt, None, 0.0, 0, -1, s)
        st()
        us = timed(st, 20)
        E = mesh.n_triangles
        blocks = (E + 127) // 128
        print(f"N={n} E={E} blocks={blocks} waves(3/SM)={blocks / 444:.2f} {us:8.2f} us  "
              f"{us / E * 1e3:.4f} ns/elem", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [216, 224, 232, 238, 240, 244, 248, 252, 256, 262, 268])
