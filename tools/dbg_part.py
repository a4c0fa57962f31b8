"""Diagnostic: partitioned (LocalMultiRunner) vs single-domain GPU runs,
per step: max difference and which elements (interior / cut-adjacent) differ."""
import sys; sys.path.insert(0, '/root/repo')  # noqa: E702
import numpy as np
from paper_1904_08684_b200 import distributed as D, mesh as M, scenario as S
from paper_1904_08684_b200.solver import Discretization

cases = [(4, "walls", "blocks", "gather"), (4, "walls", "strips", "gather"), (4, "mms", "strips", "gather"),
         (3, "walls", "blocks", "gather")]
for k, case, part, tr in cases:
    n = 16
    mesh = M.build_unit_square_mesh(n)
    scn = S.mms_scenario(dt=1e-4) if case == "mms" else S.bump_scenario(seed=0, dt=2e-4, cfl=None)
    disc = Discretization(mesh, scn, k)
    p = {"strips": D.strip_partition(n, 4), "blocks": D.block_partition(n, 2, 2)}[part]
    run = D.LocalMultiRunner(mesh, scn, k, p, transport=tr)
    st = disc.project_initial()
    cut = np.zeros(mesh.n_triangles, bool)
    for pr in run.parts:
        cut[pr.halo.elements[pr.halo.n_int:pr.halo.n_own]] = True
    for step in range(4):
        got = np.zeros_like(st.c)
        for ids, c in run.owned_state():
            got[ids] = c
        d = np.abs(got - st.c).max(axis=(1, 2))
        print(k, case, part, tr, "step", step, "max", d.max(), "diff elems: cut", int((d[cut] > 0).sum()),
              "interior", int((d[~cut] > 0).sum()), flush=True)
        st = disc.step(st)
        run.step()
