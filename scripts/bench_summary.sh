#!/bin/bash
# usage: scripts/bench_summary.sh <workload> [extra bench args]
w=$1; shift
timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --also "" "$@" 2>&1 | python -c "
import json,sys
lines=sys.stdin.read().strip().splitlines()
try:
    d=json.loads(lines[-1]); r=d['roofline']
    print(d['config']['workload'], 'samples/s', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'mainTF', round(r['achieved']), 'frac', round(r['frac'],3), 'main_ms', round(r['avg_launch_ms'],3), 'share', round(r['main_kernel_share_of_step'],3), 'e2e', round(d['e2e']['value']), 'clk', d.get('clocks'))
except Exception as e:
    print('FAILED', e); print('\n'.join(lines[-15:]))
"
