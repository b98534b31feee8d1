"""Summarise a round's ncu outputs (from scripts/profile_round.sh) into profiles/.

usage: python scripts/summarize_ncu.py <workload> <round tag, e.g. r01b>
  gpurun_out/launches_<w>.csv  -> profiles/<tag>_launches_<w>.csv   (per-kernel shares of the timed steps)
  gpurun_out/prof_<w>.ncu-rep  -> profiles/<tag>_ncu_main_<w>.txt   (key metrics of one fused-kernel launch)
                                  profiles/ncu_main_<w>.json        (read by bench.py: DRAM bytes per launch)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
w, tag = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "profiles")

# ---- launch list
rows = [l for l in open(os.path.join(ROOT, "gpurun_out", f"launches_{w}.csv")) if l.startswith('"')]
rd = list(csv.DictReader(io.StringIO("".join(rows))))
per = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for r in rd:
    k = r["Kernel Name"].split("(")[0].split("<")[0].strip()
    per[k][r["Metric Name"]] += float(r["Metric Value"].replace(",", ""))
    ids[k].add(r["ID"])
tot = sum(v["gpu__time_duration.sum"] for v in per.values())
with open(os.path.join(out, f"{tag}_launches_{w}.csv"), "w") as f:
    f.write(f"# ncu --nvtx-include timed_steps/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
            f"dram__bytes_write.sum --clock-control none: the timed steps of `bench.py --workload {w} --steps 3`\n")
    f.write("# cold-cache, serialised per-launch times: compare SHARES, not absolutes\n")
    f.write("kernel,launches,avg_us,share_of_step,dram_read_MB_per_launch,dram_write_MB_per_launch,achieved_GBps\n")
    for k, v in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        n = len(ids[k])
        t = v["gpu__time_duration.sum"] / n  # ns
        rb, wb = v["dram__bytes_read.sum"] / n, v["dram__bytes_write.sum"] / n
        f.write(f"{k},{n},{t / 1e3:.1f},{v['gpu__time_duration.sum'] / tot:.4f},{rb / 1e6:.2f},{wb / 1e6:.2f},"
                f"{(rb + wb) / t:.0f}\n")
print(open(os.path.join(out, f"{tag}_launches_{w}.csv")).read())

# ---- full capture of the fused kernel
if "--launches-only" in sys.argv:
    sys.exit(0)
rep = os.path.join(ROOT, "gpurun_out", f"prof_{w}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], rr[2]
m = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
want = [
    ("gpu__time_duration.sum", "cold-cache, serialised"),
    ("sm__cycles_active.avg", ""),
    ("dram__bytes_read.sum", "pool read once per launch"),
    ("dram__bytes_write.sum", "segment partials"),
    ("lts__t_sector_hit_rate.pct", "row groups share each pool tile through L2"),
    ("derived__lts__lts2xbar_bytes.sum.per_second", "L2 -> SM"),
    ("derived__lts__lts2xbar_bytes.sum.peak_sustained", ""),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tcgen05.mma (UTCHMMA) busy"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "UMMA operand reads from smem"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ""),
    ("launch__registers_per_thread", ""),
    ("launch__shared_mem_per_block_dynamic", ""),
    ("launch__grid_size", ""),
    ("launch__block_size", ""),
    ("launch__cluster_dim_x", ""),
]
lines = [f"# {tag} -- ncu --set full --clock-control none --import-source on -k regex:dcp_pc -c 1 "
         f"(first fused-kernel launch inside the timed steps)",
         f"#   command: python bench.py --workload {w} --steps 3 --warmup 3 --no-cpu-baseline --also none (N=1)"]
js = {}
for k, note in want:
    if k in m:
        v, u = m[k]
        lines.append(f"{k:<80} {v} {u}" + (f"   ({note})" if note else ""))
        js[k] = f"{v} {u}".strip()
# stall reasons of the whole kernel (warp-state samples)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
sr = list(csv.reader(io.StringIO(src)))
if len(sr) > 2:
    h2 = sr[1]
    ix = {k: i for i, k in enumerate(h2)}
    st = [k for k in h2 if k.startswith("stall_") and "Not Issued" not in k]
    tot_s = collections.Counter()
    ops = collections.Counter()
    for r in sr[2:]:
        for k in st:
            tot_s[k] += float(r[ix[k]] or 0)
        op = r[1].strip().split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            ops[o.split(".")[0]] += 1
    s = sum(tot_s.values())
    lines.append("warp-state samples (all warps): " + ", ".join(f"{k[6:]} {v / s:.1%}" for k, v in tot_s.most_common(8)))
    lines.append("SASS evidence: " + ", ".join(f"{o} x{ops[o]}" for o in ("UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP",
                                                                        "LDTM", "STTM", "FFMA2", "FADD2", "FMNMX3")
                                              if ops[o]))
open(os.path.join(out, f"{tag}_ncu_main_{w}.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
dr = float(m["dram__bytes_read.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1}[m["dram__bytes_read.sum"][1]]
dw = float(m["dram__bytes_write.sum"][0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[m["dram__bytes_write.sum"][1]]
rec = {"kernel": "dcp_pc_kernel", "workload": w, "tag": tag, "dram_bytes_per_launch": dr + dw,
       "dram_read_bytes": dr, "dram_write_bytes": dw, "metrics": js,
       "source": f"ncu --set full --clock-control none ({tag}, gpurun_out/prof_{w}.ncu-rep)"}
# the counters-only pass over 10 timed launches (profile_round.sh): its median is the per-launch figure
dv = os.path.join(ROOT, "gpurun_out", f"dramvar_{w}.csv")
if os.path.exists(dv):
    rows = [l for l in open(dv) if l.startswith('"')]
    per_id = collections.defaultdict(dict)
    for r in csv.DictReader(io.StringIO("".join(rows))):
        per_id[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    tot_b = sorted(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in per_id.values())
    med = tot_b[len(tot_b) // 2]
    rec.update({"dram_bytes_set_full": dr + dw, "dram_bytes_per_launch": med, "dram_bytes_launches": tot_b,
                "source": f"median of {len(tot_b)} timed launches, ncu --metrics dram__bytes_read.sum,"
                          f"dram__bytes_write.sum --clock-control none ({tag}); dram_bytes_set_full: the "
                          f"--set full capture (gpurun_out/prof_{w}.ncu-rep)"})
    with open(os.path.join(out, f"{tag}_ncu_main_{w}.txt"), "a") as f:
        f.write(f"DRAM bytes per launch, counters-only pass over {len(tot_b)} timed launches: median "
                f"{med / 1e9:.3f} GB (min {tot_b[0] / 1e9:.3f}, max {tot_b[-1] / 1e9:.3f})\n")
json.dump(rec, open(os.path.join(out, f"ncu_main_{w}.json"), "w"), indent=1)
