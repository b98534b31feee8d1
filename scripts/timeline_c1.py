"""Per-kernel device timeline of a few bench steps (torch.profiler / CUPTI, no nsys in the image):
kernel durations, and the idle gaps between consecutive kernels of the head's stream.

usage (under gpurun): python scripts/timeline_c1.py [workload] [steps] [ema_overlap]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2105_10375_b200 as dcp  # noqa: E402
import synth  # noqa: E402


def main():
    w = sys.argv[1] if len(sys.argv) > 1 else "c1"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    overlap = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    cfg = bench._workload(w)
    dev = torch.device("cuda", 0)
    M, N_loc, d = cfg.M_loc, cfg.N_loc(), cfg.d
    head = dcp.DCPHead(cfg.C, d, dcp.BF16, 1, 0, n_local_max=N_loc, m_local_max=M, device=dev)
    stream = torch.cuda.Stream(device=dev, priority=-1)
    side = torch.cuda.Stream(device=dev, priority=0)
    torch.cuda.set_stream(stream)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    for b in range(cfg.prefill_blocks()):
        gb = torch.randn(M, d, device=dev, generator=gen)
        head.enqueue((gb / gb.norm(dim=-1, keepdim=True)).bfloat16(), torch.randint(0, cfg.n_id, (M,), device=dev, generator=gen))
    ins = []
    for t in range(4):
        s = synth.step_inputs(cfg, t)
        ins.append((torch.from_numpy(s.x.view(np.int16)).view(torch.bfloat16).to(dev), torch.from_numpy(s.y).to(dev),
                    torch.from_numpy(s.pairing).to(dev), torch.from_numpy(s.g.view(np.int16)).view(torch.bfloat16).to(dev),
                    torch.from_numpy(s.gy).to(dev)))
    p = torch.randn(bench.EMA_PARAMS, device=dev) * 0.05
    g = torch.randn(bench.EMA_PARAMS, device=dev) * 0.05
    dx = torch.empty(N_loc, d, dtype=torch.bfloat16, device=dev)
    loss = torch.zeros((), device=dev)
    ev = torch.cuda.Event()

    def step(i):
        x, y, pr, gg, gy = ins[i % 4]
        head.enqueue(gg, gy)
        head.loss_fwd_bwd(x, y, pr, cfg.s, cfg.m, dx=dx, loss=loss)
        if overlap:
            ev.record(stream)
            side.wait_event(ev)
            dcp.gnet_ema(p, g, 0.999, stream=side)
        else:
            dcp.gnet_ema(p, g, 0.999)

    for i in range(5):
        step(i)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(steps):
            step(i)
        stream.wait_stream(side)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0 and "Memcpy" not in e.name
           and "Memset" not in e.name]
    evs.sort(key=lambda e: e.time_range.start)
    rows = [(e.name.split("(")[0].split("<")[0].replace("void ", "").replace("f2c::", ""), e.time_range.start,
             e.time_range.end) for e in evs]
    t0, t1 = rows[0][1], max(r[2] for r in rows)
    head_rows = [r for r in rows if not r[0].startswith("k_ema")]
    per = {}
    for n, a, b in rows:
        per.setdefault(n, []).append(b - a)
    gaps = [head_rows[i + 1][1] - head_rows[i][2] for i in range(len(head_rows) - 1)]
    out = {"workload": w, "steps": steps, "ema_overlap": overlap, "us_per_step": (t1 - t0) / steps,
           "kernels_us_mean": {k: float(np.mean(v)) for k, v in per.items()},
           "head_stream_busy_us_per_step": sum(b - a for _, a, b in head_rows) / steps,
           "head_gap_us_per_step": float(sum(max(0.0, x) for x in gaps)) / steps,
           "head_gap_us_median": float(np.median([max(0.0, x) for x in gaps]))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
