"""Per-tile timestamps of cluster 0 of dcp_pc4_kernel (debug hook; each CTA its own SM clock)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2105_10375_b200 as dcp
from paper_2105_10375_b200.dcp import load_library
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
import synth
from bench import _workload
cfg = _workload(wl)
L = load_library()
K = int(os.environ.get("F2C_TL_K", "1"))
head = dcp.DCPHead(cfg.C, cfg.d, 0, 1, 0, n_local_max=cfg.N_loc(), m_local_max=cfg.M_loc, K=K)
if os.environ.get("F2C_TL_LCOS"):  # e.g. "2,0,1" (NEXT-3 max)
    m_, h_, l_ = os.environ["F2C_TL_LCOS"].split(",")
    head.set_lcos(int(m_), bool(int(h_)), float(l_))
gen = torch.Generator(device="cuda"); gen.manual_seed(1)
for b in range(cfg.prefill_blocks()):
    g = torch.randn(cfg.M_loc, K, cfg.d, device="cuda", generator=gen) if K > 1 else torch.randn(cfg.M_loc, cfg.d, device="cuda", generator=gen)
    g = (g / g.norm(dim=-1, keepdim=True)).bfloat16()
    head.enqueue(g, torch.randint(0, cfg.n_id, (cfg.M_loc,), device="cuda", generator=gen))
st = synth.step_inputs(cfg, 0)
x = torch.from_numpy(st.x.view(np.int16)).view(torch.bfloat16).cuda()
y = torch.from_numpy(st.y).cuda(); pr = torch.from_numpy(st.pairing).cuda()
gk = np.stack([st.g] * K, axis=1) if K > 1 else st.g
head.enqueue(torch.from_numpy(np.ascontiguousarray(gk).view(np.int16)).view(torch.bfloat16).cuda(), torch.from_numpy(st.gy).cuda())
buf = torch.zeros(64 * 16 + 64, dtype=torch.int64, device="cuda")
L.f2c_dcp_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for it in range(3):
    head.loss_fwd_bwd(x, y, pr, 64, 0.35)
L.f2c_dcp_debug_timestamps(head._h, ctypes.c_void_p(buf.data_ptr()))
head.loss_fwd_bwd(x, y, pr, 64, 0.35)
torch.cuda.synchronize()
bb = buf.cpu().numpy().astype(np.int64)
a = bb[:1024].reshape(64, 16)
names = {0: "PL g1 start", 1: "PL sempty ok", 2: "PL g1 issued", 3: "PL sfull seen", 4: "PL pready",
         5: "PL mv pready", 6: "PL mv slotfree", 7: "PL mv copied", 8: "CL pfull", 9: "CL pfull_peer",
         10: "CL g2 issued", 11: "CP pfull", 12: "PL sm ld done", 13: "PL sm compute done", 14: "PL sm sempty arrived",
         15: "PL sm pstage ok"}
ntl = int((a[:, 0] > 0).sum())
print("tiles recorded", ntl)
PL = [0, 1, 2, 3, 12, 13, 15, 4, 5, 6, 7]
CL = [8, 9, 10]
for j in range(min(ntl, int(os.environ.get("F2C_TL_ROWS", "20")))):
    print(j, "PL", [int(a[j, k] - a[0, 0]) for k in PL], "CL", [int(a[j, k] - a[0, 8]) for k in CL], "CP", int(a[j, 11] - a[0, 11]))
lo, hi = 8, min(ntl, 60)
for k in sorted(names):
    d = np.diff(a[lo:hi, k])
    print("cadence %-16s median %7.0f" % (names[k], np.median(d)))
def lat(k1, k0):
    return np.median(a[lo:hi, k1] - a[lo:hi, k0])
print("PL softmax: sfull->ld done %.0f, ld->arrived %.0f, ->compute done %.0f, pstage wait %.0f, P write+arrive %.0f" % (lat(12, 3), lat(14, 12), lat(13, 14), lat(15, 13), lat(4, 15)))
print("PL: sempty wait %.0f, g1 issue %.0f; sfull seen - g1 issued %.0f; softmax (sfull->pready) %.0f" % (lat(1, 0), lat(2, 1), lat(3, 2), lat(4, 3)))
print("PL mover: pready->slotfree %.0f, copy %.0f" % (lat(6, 5), lat(7, 6)))
print("CL: pfull -> pfull_peer %.0f, -> issued %.0f" % (lat(9, 8), lat(10, 9)))
spans = bb[1024:1056]
print("cluster spans (cycles):", spans[spans > 0].tolist())
print("cluster spans (ns, clusters 0-7):", bb[1056:1064].tolist(), " -> MHz", (spans[:8] / np.maximum(bb[1056:1064], 1) * 1e3).round().tolist())
head.profile(True)
for it in range(20):
    head.loss_fwd_bwd(x, y, pr, 64, 0.35)
torch.cuda.synchronize()
ms, nl, npos = head.profile_read()
print("profiled fused-kernel ms per launch: %.3f over %d launches" % (ms / max(nl, 1), nl))
