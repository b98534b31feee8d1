#!/bin/bash
# The tail role (F2C_TAIL=0 off / 1 forced, F2C_TAIL_TAU = the schedule's cost of a tail tile) at c3 and c1.
# usage (under gpurun): bash scripts/ab_tail.sh "0:0.6 1:0.6 1:0.8" "c3 c1"
out=gpurun_out/tail_summary.txt
rm -f $out
for pass in 1 2; do
  for v in $1; do
    M=${v%%:*}; T=${v##*:}
    for W in $2; do
      F2C_TAIL=$M F2C_TAIL_TAU=$T python bench.py --workload $W --also none --no-cpu-baseline --no-w-parity --steps 20 --warmup 5 --trials 1 > gpurun_out/tl.json 2>&1
      python -c "
import json; d=json.loads(open('gpurun_out/tl.json').read().strip().splitlines()[-1]); r=d['roofline']
print('tail=$M tau=$T', '$W', round(d['ms_per_step'],4), 'launch', round(r['avg_launch_ms'],4), 'fb', round(r['frac_vs_burst'],3), d['clocks']['sm_mhz'])" >> $out 2>&1
    done
  done
done
cat $out
