#!/bin/bash
# A/B of library builds: short (10-step) and sustained (200-step) c3 timings plus the fused kernel's DRAM
# bytes per launch (ncu, one launch).  usage (under gpurun): LIBS="lib_a lib_b" bash scripts/ab_dram.sh
out=gpurun_out/abd_summary.txt
rm -f $out
for pass in 1 2; do
  for L in $LIBS; do
    for W in ${WLS:-c3}; do
      F2C_LIB=ab/$L.so python bench.py --workload $W --also none --no-cpu-baseline --no-w-parity --steps 10 --warmup 3 --trials 1 > gpurun_out/abd_${L}_$W.json 2>&1
      python -c "
import json; d=json.loads(open('gpurun_out/abd_${L}_$W.json').read().strip().splitlines()[-1]); r=d['roofline']
print('short $L $W', round(d['ms_per_step'],3), 'launch', round(r['avg_launch_ms'],3), d['clocks']['sm_mhz'])" >> $out 2>&1
    done
    F2C_LIB=ab/$L.so python bench.py --workload c3 --also none --no-cpu-baseline --no-w-parity --steps 200 --warmup 5 --trials 1 > gpurun_out/abd_${L}_sus.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/abd_${L}_sus.json').read().strip().splitlines()[-1]); r=d['roofline']
print('sustained $L c3', round(d['ms_per_step'],3), 'launch', round(r['avg_launch_ms'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))" >> $out 2>&1
  done
done
for L in $LIBS; do
  F2C_LIB=ab/$L.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:dcp_pc_kernel -s 3 -c 1 --csv python bench.py --workload c3 --also none --no-cpu-baseline --no-w-parity --steps 2 --warmup 3 --trials 1 \
    > gpurun_out/abd_${L}_ncu.csv 2>&1
  echo "ncu $L: $(grep -E 'dram__bytes_read.sum|dram__bytes_write.sum|gpu__time_duration' gpurun_out/abd_${L}_ncu.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | tr '\n' ' ')" >> $out
done
cat $out
