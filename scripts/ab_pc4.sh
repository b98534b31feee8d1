# A/B of the fused kernels (F2C_KERNEL=pc: CTA pairs, 128-row groups; pc4: 2-SM pairs, 256-row groups)
for w in ${@:-c3 c2 c3r_8 c1}; do
  for k in pc pc4 pc pc4; do
    r=$(F2C_KERNEL=$k timeout 300 python bench.py --workload $w --steps 60 --warmup 5 --no-cpu-baseline --also none 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g samples/s  frac %.3f  kernel_ms %.3f  N_pos %.0f  clk %s' % (d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['roofline']['N_pos_avg'], d['clocks']['sm_mhz']))")
    echo "$w $k: $r"
  done
done
