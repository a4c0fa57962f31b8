import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1904_08684_b200 import distributed as D, mesh as M, scenario as S
from paper_1904_08684_b200.solver import Discretization
for k, case, part in [(3, "walls", "blocks"), (3, "walls", "strips"), (2, "walls", "blocks"), (3, "mms", "strips"), (4, "walls", "blocks")]:
    n, steps = 16, 4
    mesh = M.build_unit_square_mesh(n)
    scn = S.mms_scenario(dt=1e-4) if case == "mms" else S.bump_scenario(seed=0, dt=2e-4, cfl=None)
    disc = Discretization(mesh, scn, k)
    out = disc.run(disc.project_initial(), t_end=steps * scn.dt)
    p = {"strips": D.strip_partition(n, 4), "blocks": D.block_partition(n, 2, 2)}[part]
    run = D.LocalMultiRunner(mesh, scn, k, p)
    for _ in range(steps):
        run.step()
    got = np.zeros_like(out.c)
    for ids, c in run.owned_state():
        got[ids] = c
    d = np.abs(got - out.c)
    print(k, case, part, "max abs diff", d.max(), "rel", d.max() / np.abs(out.c).max(), "n elems differing", int((d.max(axis=(1,2)) > 0).sum()))
