#!/bin/bash
# ncu launch lists (per-kernel device time of the timed steps) for several workloads, ONE GPU.
# usage (under gpurun): bash scripts/launch_lists.sh c4r_1_16384 c4r_10_2048 ...
# Post-process here: python scripts/summarize_ncu.py <w> <tag> --launches-only
for W in "$@"; do
  CMD="python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --also none --trials 1 --no-w-parity"
  ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/ncu_l_$W.log 2>&1
done
