"""Per-tile timestamps of CTA 0 of the fused kernel (debug build hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_10375_b200 as dcp
from paper_2105_10375_b200.dcp import load_library
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
import synth
cfg = synth.CONFIGS[wl]
L = load_library()
head = dcp.DCPHead(cfg.C, cfg.d, 0, 1, 0, n_local_max=cfg.N_loc(), m_local_max=cfg.M_loc)
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for b in range(cfg.prefill_blocks()):
    g = torch.randn(cfg.M_loc, cfg.d, device="cuda", generator=gen); g = (g / g.norm(dim=1, keepdim=True)).bfloat16()
    head.enqueue(g, torch.randint(0, cfg.n_id, (cfg.M_loc,), device="cuda", generator=gen))
st = synth.step_inputs(cfg, 0)
x = torch.from_numpy(st.x.view(np.int16)).view(torch.bfloat16).cuda()
y = torch.from_numpy(st.y).cuda(); pr = torch.from_numpy(st.pairing).cuda()
head.enqueue(torch.from_numpy(st.g.view(np.int16)).view(torch.bfloat16).cuda(), torch.from_numpy(st.gy).cuda())
buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
L.f2c_dcp_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for it in range(3):
    head.loss_fwd_bwd(x, y, pr, 64, 0.35)
L.f2c_dcp_debug_timestamps(head._h, ctypes.c_void_p(buf.data_ptr()))
head.loss_fwd_bwd(x, y, pr, 64, 0.35)
torch.cuda.synchronize()
a = buf.view(64, 8).cpu().numpy().astype(np.int64)
t0 = a[0, 0]
print("cols: mma_g1_start g1_issued pfull_done g2_issued | epi_wait_start sfull_done pfull_arrive | prod_lastpair_issue (rel cycles)")
for j in range(40):
    r = a[j] - t0
    print(j, r.tolist(), " tile:", (a[j + 1, 0] - a[j, 0]) if j < 63 else 0)
d = np.diff(a[:40, 0])
print("median cycles per tile", np.median(d))
print("median g1 issue", np.median(a[:40, 1] - a[:40, 0]), "median sfull->pfull(epi)", np.median(a[:40, 6] - a[:40, 5]),
      "median g1_issued->pfull_done(mma)", np.median(a[:40, 2] - a[:40, 1]), "median g2 issue", np.median(a[:40, 3] - a[:40, 2]),
      "median epi sfull wait", np.median(a[:40, 5] - a[:40, 4]))
