#!/bin/bash
# dcp_pc4_kernel with the multi-wave range schedule (k_compact) vs dcp_pc_kernel, and vs pc4 with the
# round-1 single-wave rule (ab/lib_ref.so).  usage (under gpurun): bash scripts/ab_pc4w.sh "c3r_8 c4r_10_16384"
out=gpurun_out/pc4w_summary.txt
rm -f $out
WLS="$1"
for pass in 1 2; do
  for w in $WLS; do
    for v in "lib_pc4w pc" "lib_pc4w pc4" "lib_ref pc4"; do
      set -- $v
      F2C_LIB=ab/$1.so F2C_KERNEL=$2 timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --trials 1 --no-cpu-baseline --no-w-parity --also none > gpurun_out/pc4w.json 2>&1
      python -c "
import json; d=json.loads(open('gpurun_out/pc4w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', '$1', '$2', round(d['ms_per_step'],4), 'launch', round(r['avg_launch_ms'],4), 'fb', round(r['frac_vs_burst'],3), d['clocks']['sm_mhz'])" >> $out 2>&1
    done
  done
done
cat $out
