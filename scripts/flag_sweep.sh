#!/bin/bash
# timing experiments: which part of dcp_pc_kernel bounds it (results are void under flags)
for f in 0 4 8 12 16 20 28 1; do
  F2C_DBG_FLAGS=$f python bench.py --workload ${1:-c2} --also "" --no-cpu-baseline --steps 60 --warmup 3 2>/dev/null \
   | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('flags', $f, 'kernel ms %.3f' % r['avg_launch_ms'], 'TF %.0f' % r['achieved'], j['clocks']['sm_mhz'])"
done
