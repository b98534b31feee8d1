CMD="python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --also none --trials 1 --no-w-parity"
timeout 600 ncu --nvtx --nvtx-include "timed_steps/" -k regex:dcp_pc_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file gpurun_out/dramvar_c3.csv $CMD > gpurun_out/dramvar.log 2>&1
CMD="python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline --also none --trials 1 --no-w-parity"
timeout 600 ncu --nvtx --nvtx-include "timed_steps/" -k regex:dcp_pc_kernel --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file gpurun_out/dramvar_c2.csv $CMD >> gpurun_out/dramvar.log 2>&1
grep -E "dram__bytes_read|duration" gpurun_out/dramvar_c3.csv | awk -F'","' '{print $(NF-2), $NF}' | head -30
