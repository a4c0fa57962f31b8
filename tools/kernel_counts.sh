#!/bin/bash
# usage (GPU box): tools/kernel_counts.sh c2 c3 c4 c5  -> gpurun_out/counts_<cfg>.csv
M=$(python -c "import sys; sys.path.insert(0,'tools'); import kernel_counts as k; print(k.METRICS)")
for c in "$@"; do
  python tools/kernel_counts.py $c > gpurun_out/counts_$c.log 2>&1 || { echo "$c failed"; continue; }
  ncu --nvtx --nvtx-include "measure/" --metrics $M --clock-control none --csv \
      --log-file gpurun_out/counts_$c.csv python tools/kernel_counts.py $c >> gpurun_out/counts_$c.log 2>&1
done
