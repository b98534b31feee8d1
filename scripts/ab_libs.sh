for L in ${LIBS:-lib_1b0c2e2 lib_wt2}; do
  for W in ${WLS:-c3r_8 c3 c2}; do
    F2C_LIB=ab/$L.so python bench.py --workload $W --also none --no-cpu-baseline --no-w-parity --steps 10 --warmup 3 --trials 1 > gpurun_out/ab_${L}_$W.json 2>&1
    python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_${L}_$W.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$L', '$W', round(d['ms_per_step'],3), 'launch', round(r['avg_launch_ms'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_summary.txt 2>&1
  done
done
