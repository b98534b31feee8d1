"""Host-side cost of one bench step (Python binding + library host code + launches) against its
device time: if the host needs longer per step than the GPU, the step is host-bound.
usage (under gpurun): python scripts/host_overhead.py [workload] [steps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2105_10375_b200 as dcp  # noqa: E402
import synth  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = bench._workload(w)
dev = torch.device("cuda", 0)
M, N_loc, d = cfg.M_loc, cfg.N_loc(), cfg.d
head = dcp.DCPHead(cfg.C, d, dcp.BF16, 1, 0, n_local_max=N_loc, m_local_max=M, device=dev)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
for b in range(cfg.prefill_blocks()):
    gb = torch.randn(M, d, device=dev, generator=gen)
    head.enqueue((gb / gb.norm(dim=-1, keepdim=True)).bfloat16(), torch.randint(0, cfg.n_id, (M,), device=dev, generator=gen))
s = synth.step_inputs(cfg, 0)
x = torch.from_numpy(s.x.view(np.int16)).view(torch.bfloat16).to(dev)
y, pr = torch.from_numpy(s.y).to(dev), torch.from_numpy(s.pairing).to(dev)
gg = torch.from_numpy(s.g.view(np.int16)).view(torch.bfloat16).to(dev)
gy = torch.from_numpy(s.gy).to(dev)
p = torch.randn(bench.EMA_PARAMS, device=dev) * 0.05
g = torch.randn(bench.EMA_PARAMS, device=dev) * 0.05
dx = torch.empty(N_loc, d, dtype=torch.bfloat16, device=dev)
loss = torch.zeros((), device=dev)
out = {}
for mode in ("full", "no_ema"):
    for _ in range(5):
        head.enqueue(gg, gy)
        head.loss_fwd_bwd(x, y, pr, cfg.s, cfg.m, dx=dx, loss=loss)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(K):
        head.enqueue(gg, gy)
        head.loss_fwd_bwd(x, y, pr, cfg.s, cfg.m, dx=dx, loss=loss)
        if mode == "full":
            dcp.gnet_ema(p, g, 0.999)
    t_host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    out[mode] = {"host_us_per_step": 1e6 * t_host / K, "device_us_per_step": 1e3 * e0.elapsed_time(e1) / K}
# the calls alone (host side of each entry point)
for name, fn in (("enqueue", lambda: head.enqueue(gg, gy)),
                 ("loss_fwd_bwd", lambda: head.loss_fwd_bwd(x, y, pr, cfg.s, cfg.m, dx=dx, loss=loss)),
                 ("gnet_ema", lambda: dcp.gnet_ema(p, g, 0.999))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    out[f"host_us_{name}"] = 1e6 * (time.perf_counter() - t0) / 50
    torch.cuda.synchronize()
print(json.dumps({"workload": w, **out}, indent=1))
