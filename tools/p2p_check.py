"""Multi-process check of the p2p halo transport (CUDA IPC + stream flags +
fused push) against the single-domain run.  Launch:

    torchrun --standalone --nproc-per-node 2 tools/p2p_check.py [k] [steps] [n] [graph] [blocks] [mms]

graph = 1 (default): every rank replays its step as one captured CUDA graph
(qf_graph_*: stage launches, flag waits / writes, both streams); blocks = 1:
px x py block partition instead of strips; mms = 1: the manufactured
solution (time-dependent Dirichlet data and forcing, device time).

Uses a gloo process group (host objects only: IPC handles, recv lists) so
that it also runs with several ranks on one GPU; no kernel waits on another
(ordering by stream memory operations)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1904_08684_b200 import distributed as D, mesh as M, scenario as S  # noqa: E402


def main(k=2, steps=3, n=16, graph=1, blocks=0, mms=0):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    mesh = M.build_unit_square_mesh(n)
    scn = S.mms_scenario(dt=2e-4) if mms else S.bump_scenario(seed=0, dt=2e-4, cfl=None)
    part = D.block_partition(n, *D.block_shape(world)) if blocks else D.strip_partition(n, world)
    run = D.DistributedRunner(mesh, scn, k, part, rank, world, transport="p2p", graph=bool(graph))
    if mms and not graph:
        run.use_device_time()  # same time arithmetic as the single-domain run
    for _ in range(steps):
        run.step()
    run.sync()
    torch.cuda.synchronize()
    nown = run.halo.n_own
    mine = (run.halo.elements[:nown], run.c[:, :, :nown].permute(2, 0, 1).cpu().numpy())
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank == 0:
        from paper_1904_08684_b200.solver import Discretization
        disc = Discretization(mesh, scn, k)
        ref = disc.run(disc.project_initial(), t_end=steps * scn.dt).c
        out = np.zeros_like(ref)
        for ids, c in got:
            out[ids] = c
        how = "graph" if run._graph is not None else f"eager ({getattr(run, 'graph_note', 'graph off')})"
        print(f"p2p world={world} k={k} steps={steps} n={n} {'blocks' if blocks else 'strips'} "
              f"{'mms' if mms else 'bumps'} [{how}] transport={run.transport}: bit-identical to single domain: "
              f"{np.array_equal(out, ref)} (max diff {np.abs(out - ref).max():.3e})", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
