"""Diagnostic: stage-kernel time vs the number of elements updated (qf_stage
on a sub-range), to expose wave quantisation; C2 problem (MMS, k = 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1904_08684_b200 import mesh as M, scenario as S  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402
from tools.term_timing import timed  # noqa: E402


def main(k=2, n=256):
    mesh = M.build_unit_square_mesh(n)
    disc = Discretization(mesh, S.mms_scenario(dt=2e-5), k)
    ds = disc.to_device(disc.project_initial())
    lib, s = disc._lib, torch.cuda.current_stream().cuda_stream
    w = disc._work_buf()
    lib.qf_ghost(disc._ctx, 0.0, s)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    E = mesh.n_triangles
    for ne in sorted({E, E // 2, E // 4, sms * 128, sms * 256, sms * 384, sms * 384 * 2, sms * 768,
                      sms * 512, sms * 128 * 5, sms * 128 * 7}):
        if ne > E:
            continue
        st = lambda: lib.qf_stage(disc._ctx, ds.c.data_ptr(), ds.u.data_ptr(), ds.c.data_ptr(),  # noqa
                                  w.data_ptr(), w[3 * disc.K * disc.ld:].data_ptr(), 0.5, 0.5,
                                  0.0, disc.dt, None, 0.0, 0, ne, s)
        st()
        us = timed(st, 20)
        print(f"k={k} n={ne:7d} ({ne / (sms * 128):5.2f} blocks/SM): {us:8.1f} us  {us / ne * 1e3:6.3f} ns/elem")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
