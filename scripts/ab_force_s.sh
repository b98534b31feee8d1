#!/bin/bash
# Timing experiment: the fused kernel's range count S forced (F2C_FORCE_S) against the default schedule.
# usage (under gpurun): bash scripts/ab_force_s.sh "c3r_8:0 c3r_8:13 c3:0 c3:29 c3:59"
for p in $1; do
  W=${p%%:*}; S=${p##*:}
  F2C_FORCE_S=$S python bench.py --workload $W --also none --no-cpu-baseline --no-w-parity --steps 10 --warmup 3 --trials 2 > gpurun_out/fs_${W}_$S.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/fs_${W}_$S.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$W S=$S', round(d['ms_per_step'],3), 'launch', round(r['avg_launch_ms'],3), d['clocks']['sm_mhz'])" >> gpurun_out/fs_summary.txt 2>&1
done
cat gpurun_out/fs_summary.txt
