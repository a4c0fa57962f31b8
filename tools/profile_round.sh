#!/bin/bash
# Round profiling on the GPU box -> gpurun_out/ (summaries only; reports stay in /tmp)
#   tools/profile_round.sh r02
R=${1:-r02}
O=gpurun_out
# 1. launch list of the default bench command (C2), cold-cache serialised per-launch times
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${R}_c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu > $O/${R}_ncu_bench.log 2>&1
python tools/launch_summary.py $O/${R}_c2_launches.csv "# ncu launch list: python bench.py --steps 2 --warmup 3 (C2)" > $O/${R}_c2_launch_summary.txt
# 2. full capture of the C2 stage kernel (first stage of an L2-flushed step)
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" -k regex:stage_kernel -c 1 \
    -o /tmp/${R}_c2_stage -f python tools/kernel_counts.py c2 > $O/${R}_c2_full.log 2>&1
python tools/ncu_summary.py /tmp/${R}_c2_stage.ncu-rep > $O/${R}_c2_stage_kernel_ncu.txt 2>&1
python tools/ncu_regions.py /tmp/${R}_c2_stage.ncu-rep 2 >> $O/${R}_c2_stage_kernel_ncu.txt 2>&1
# 3. per-kernel FP64 FLOP and DRAM bytes per element per stage, every config
tools/kernel_counts.sh c2 c3 c4 c5
for c in c2 c3 c4 c5; do
  python - $c >> $O/${R}_kernel_counts.txt 2>&1 <<PY
import sys, bench
c = sys.argv[1]
k, n, mesh, scn = bench.build_problem(c)
print(f"== {c}: k={k} n={n} E={mesh.n_triangles}")
import subprocess
print(subprocess.run([sys.executable, "tools/kernel_counts.py", "--parse", f"gpurun_out/counts_{c}.csv",
                      str(mesh.n_triangles), str(bench.stages_of(k))], capture_output=True, text=True).stdout)
PY
done
# 4. full captures of the k = 3, 4 kernels of one stage (walls, N = 512)
for k in 3 4; do
  ncu --set full --clock-control none -k regex:"stage_kernel|volume_kernel|velocity_kernel" --launch-skip 2 -c 4 \
      -o /tmp/${R}_k$k -f python tools/order_timing.py 512 --orders $k --once > $O/${R}_k${k}_full.log 2>&1
  python tools/ncu_summary.py /tmp/${R}_k$k.ncu-rep > $O/${R}_k${k}_kernels_ncu.txt 2>&1
done
# 4b. full capture of the C4 stage kernel (p = 2, walls, jittered mesh, 8.4M elements: the config HBM could bind)
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "measure/" -k regex:stage_kernel -c 1 \
    -o /tmp/${R}_c4_stage -f python tools/kernel_counts.py c4 > $O/${R}_c4_full.log 2>&1
python tools/ncu_summary.py /tmp/${R}_c4_stage.ncu-rep > $O/${R}_c4_stage_kernel_ncu.txt 2>&1
python tools/ncu_regions.py /tmp/${R}_c4_stage.ncu-rep 2 >> $O/${R}_c4_stage_kernel_ncu.txt 2>&1
# 5. setup time of C5 strong (33.5M elements) with the device-side mesh setup
python tools/setup_time.py 4096 4 > $O/${R}_setup_time_c5_strong.json 2> $O/${R}_setup_time.err
# 6. the multi-GPU runner at world size 1 (p2p transport + per-rank step graph; nccl)
for t in p2p nccl; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$((RANDOM % 10)) \
      bench.py --gpus 1 --dist --no-cpu --no-extra --steps 100 --warmup 5 --transport $t 2>/dev/null | tail -1 > $O/${R}_bench_dist_world1_$t.json
done
ls -la $O
