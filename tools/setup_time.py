"""Setup time of a BASELINE configuration on the GPU box:
mesh generation (host: vertices + triangles), device tables (connectivity,
geometry, Z-order slots: device_setup.py), device projection of the initial
state and P1 bathymetry (qf_project), and the CFL time step.

    python tools/setup_time.py 4096 4      # C5 strong: 2 x 4096^2 elements, p = 4
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(n=4096, k=4):
    import torch

    from paper_1904_08684_b200 import mesh as M, scenario as S
    from paper_1904_08684_b200.solver import Discretization

    t0 = time.perf_counter()
    mesh = M.build_unit_square_mesh(n, lazy=True)
    t1 = time.perf_counter()
    disc = Discretization(mesh, S.bump_scenario(seed=0, cfl=0.1), k)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = disc.project_initial()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(json.dumps({"n": n, "order": k, "elements": mesh.n_triangles,
                      "mesh_s": t1 - t0, "discretization_s": t2 - t1,
                      "device_tables_s": getattr(disc, "setup_seconds", None),
                      "project_initial_and_cfl_s": t3 - t2, "total_s": t3 - t0,
                      "device_tables": disc.device_tables, "device_setup": disc.device_setup,
                      "dt": disc.dt, "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
    del st


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
