#!/bin/bash
# Round profile on ONE GPU (run under gpurun): plain run, ncu launch list of the timed steps, the fused
# kernel's DRAM bytes over 10 timed launches, and ncu --set full of one fused-kernel launch.
# Post-process here with scripts/summarize_ncu.py.
set -e
W=${1:-c3}
CMD="python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --also none --trials 1 --no-w-parity"
$CMD > gpurun_out/plain_$W.log 2>&1
ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/ncu_l_$W.log 2>&1
# DRAM bytes of the fused kernel over 10 timed launches, counters only (the figure bench.py reports as
# roofline.traffic is their median; the --set full capture below is a single launch)
CMD10="python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline --also none --trials 1 --no-w-parity"
ncu --nvtx --nvtx-include "timed_steps/" -k regex:dcp_pc_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/dramvar_$W.csv $CMD10 > gpurun_out/ncu_d_$W.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed_steps/" -k regex:dcp_pc -c 1 \
    -o gpurun_out/prof_$W $CMD > gpurun_out/ncu_f_$W.log 2>&1
