"""Run a BASELINE config for a number of steps and report errors / timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1904_08684_b200.solver import Discretization  # noqa: E402


def main(cfg, n=None, steps=20, device_setup=None):
    k, n, mesh, scn = bench.build_problem(cfg, n)
    t0 = time.perf_counter()
    disc = Discretization(mesh, scn, k, device_setup=device_setup)
    st = disc.project_initial()
    print(f"{cfg} N={n} k={k} E={mesh.n_triangles} device_setup={disc.device_setup} "
          f"dt={disc.dt:.3e} setup {time.perf_counter() - t0:.1f}s", flush=True)
    for i in range(steps):
        st = disc.run(st, t_end=st.t + disc.dt)
        if i % 5 == 0:
            c = st.c if mesh.n_triangles < 300000 else None
            print(i, st.t, None if c is None else float(np.abs(c).max()), flush=True)
            if c is not None:
                st = disc.run(disc.project_initial(), t_end=st.t) if False else st
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 20)
