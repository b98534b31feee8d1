#!/bin/bash
# Timing experiment (results void under flags): sustained c3 (200 steps) with parts of the fused kernel disabled.
# usage (under gpurun): FLAGS="0 8 4 0 8 4" bash scripts/flags_sustained.sh
out=gpurun_out/flags_sus.txt
rm -f $out
for f in $FLAGS; do
  if [ "$f" = 0 ]; then unset F2C_DBG_FLAGS; else export F2C_DBG_FLAGS=$f; fi
  python bench.py --workload c3 --also none --no-cpu-baseline --no-w-parity --steps 200 --warmup 5 --trials 1 > gpurun_out/fs_$f.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/fs_$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('flags=$f c3 sustained', round(d['ms_per_step'],3), 'launch', round(r['avg_launch_ms'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))" >> $out 2>&1
done
unset F2C_DBG_FLAGS
cat $out
