"""Per-tile timestamps of CTA 0 of the fused kernel (debug build hook)."""
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
a16 = bb[:1024].reshape(64, 16)
a = a16[:, :8]
st = bb[1024:1088].reshape(8, 8)
t0 = a[0, 0]
import os
if os.environ.get("F2C_KERNEL") == "tp64":
    for j in range(40):
        print(j, (a[j] - t0).tolist())
else:
    P = a[:, :6] - a[0, 0]; Q = a[:, 6:] - a[0, 6]
    print("producer cols: g1_start g1_issued sfull_seen pready copy_issue copy_done | consumer: pfull_seen g2_issued")
    for j in range(int(os.environ.get("F2C_TL_ROWS", "24"))):
        print(j, P[j].tolist(), Q[j].tolist())
    n = 40
    for j in range(8):
        r = st[j] - a[16 + j, 0]
        print("tile", 16 + j, "stage (wait_start, wait_done) rel g1_start:", r.tolist(), " g1_issued", a[16 + j, 1] - a[16 + j, 0])
    sp = bb[1024:1032]
    ntl = int((a16[:, 0] > 0).sum())
    pro = bb[1040:1056].reshape(2, 8)
    print("prologue stamps CTA0 rel start: units done %d, cluster sync %d, x_hat in TMEM %d, MMA saw xready %d"
          % tuple(pro[0, 1:5] - pro[0, 0]))
    print("prologue (CTA 0 start -> tile 0 GEMM-1 issue): %d cycles; tiles recorded %d" % (a[0, 0] - sp[0], ntl))
    print("epilogue (last recorded tile GEMM-1 issue -> CTA 0 end): %d cycles; consumer end - its last GEMM-2 issue: %d"
          % (sp[2] - a[ntl - 1, 0], sp[6] - a16[ntl - 1, 7]))
    for c in range(2):
        cyc, ns = sp[4 * c + 2] - sp[4 * c], sp[4 * c + 3] - sp[4 * c + 1]
        print("CTA", c, "span: %d cycles, %.3f ms, eff clock %.0f MHz" % (cyc, ns / 1e6, cyc / max(ns, 1) * 1e3))
    print("softmax: sfull->ld done", np.median(a16[:n, 8] - a16[:n, 2]), "ld->compute done", np.median(a16[:n, 9] - a16[:n, 8]),
          "pstage wait", np.median(a16[:n, 10] - a16[:n, 9]), "P write+arrive", np.median(a16[:n, 3] - a16[:n, 10]),
          "pready->next sfull", np.median(a16[1:n, 2] - a16[:n - 1, 3]))
    print("producer cadence (g1_start)", np.median(np.diff(a[:n, 0])), "consumer cadence (pfull_seen)", np.median(np.diff(a[:n, 6])))
    print("g1 issue", np.median(a[:n, 1] - a[:n, 0]), "softmax sfull->pready", np.median(a[:n, 3] - a[:n, 2]),
          "copy", np.median(a[:n, 5] - a[:n, 4]), "pready->copy issue", np.median(a[:n, 4] - a[:n, 3]),
          "g2 issue", np.median(a[:n, 7] - a[:n, 6]))
