#!/bin/bash
# usage (GPU box): tools/prof_orders.sh TAG N "2 3 4"
# one full ncu capture (source-level) of the kernels of one RK stage per order
# (bump/wall problem, N x N quads; tools/order_timing.py --once runs the stage
# twice); exports the details page and the per-line source page as CSV into
# gpurun_out/ (the .ncu-rep itself stays in /tmp: too large to bring back)
TAG=$1; N=$2; ORDERS=${3:-"2 3 4"}
for k in $ORDERS; do
  rep=/tmp/prof_${TAG}_k$k
  ncu --set full --import-source on --clock-control none \
      -k regex:"stage_kernel|volume_kernel|velocity_kernel|vstage" --launch-skip ${SKIP:-0} -c ${COUNT:-4} \
      -o $rep -f python tools/order_timing.py $N --orders $k --once \
      > gpurun_out/prof_${TAG}_k$k.log 2>&1
  ncu -i $rep.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_k${k}_details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/prof_${TAG}_k${k}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_${TAG}_k${k}_source.csv 2>/dev/null
done
ls -la gpurun_out/
