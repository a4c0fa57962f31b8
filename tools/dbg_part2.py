"""Diagnostic: k=4 single-domain qf_step vs one-partition LocalMultiRunner (qf_stage per stage)."""
import sys; sys.path.insert(0, '/root/repo')  # noqa: E702
import numpy as np
import torch
from paper_1904_08684_b200 import distributed as D, mesh as M, scenario as S
from paper_1904_08684_b200.solver import Discretization

for k in (3, 4):
    n = 16
    mesh = M.build_unit_square_mesh(n)
    scn = S.bump_scenario(seed=0, dt=2e-4, cfl=None)
    disc = Discretization(mesh, scn, k)
    st0 = disc.project_initial()
    one = D.LocalMultiRunner(mesh, scn, k, np.zeros(mesh.n_triangles, dtype=np.int64))
    st = st0
    for step in range(2):
        st = disc.step(st)
        one.step()
    (ids, c), = one.owned_state()
    got = np.zeros_like(st.c); got[ids] = c
    print(k, "qf_step vs 1-partition qf_stage: max diff", np.abs(got - st.c).max(), flush=True)
    # qf_stage on the same Discretization with the same buffers as qf_step
    ds = disc.to_device(st0)
    w = disc._work_buf()
    lib, s = disc._lib, torch.cuda.current_stream().cuda_stream
    K, ld = disc.K, disc.ld
    c1 = torch.empty_like(ds.c); u1 = torch.empty_like(ds.u); c2 = torch.empty_like(ds.c); u2 = torch.empty_like(ds.u)
    c, u = ds.c, ds.u
    for step in range(2):
        t = step * disc.dt
        lib.qf_stage(disc._ctx, c.data_ptr(), u.data_ptr(), None, c1.data_ptr(), u1.data_ptr(), 0.0, 1.0, t, disc.dt, None, 0.0, 0, -1, s)
        lib.qf_stage(disc._ctx, c1.data_ptr(), u1.data_ptr(), c.data_ptr(), c2.data_ptr(), u2.data_ptr(), 0.75, 0.25, t, disc.dt, None, 0.0, 0, -1, s)
        lib.qf_stage(disc._ctx, c2.data_ptr(), u2.data_ptr(), c.data_ptr(), c.data_ptr(), u.data_ptr(), 1/3, 2/3, t, disc.dt, None, 0.0, 0, -1, s)
    from paper_1904_08684_b200.solver import State
    st3 = State(t=0.0, _dev=(disc, ds))
    print(k, "qf_step vs qf_stage same ctx: max diff", np.abs(st3.c - st.c).max(), flush=True)
