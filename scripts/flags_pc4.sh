# timing experiments for dcp_pc4_kernel (results void): kernel ms per launch at c2 under F2C_DBG_FLAGS
for f in 0 4 8 12 128 256 512 64 768 832 972; do
  r=$(F2C_KERNEL=pc4 F2C_DBG_FLAGS=$f timeout 120 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --also none 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kernel_ms %.3f' % d['roofline']['avg_launch_ms'])" 2>&1 | tail -1)
  echo "flags $f: $r"
done
