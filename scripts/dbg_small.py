"""Quick GPU sanity run: one small case, prints GPU vs oracle numbers."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from helpers import to_dev, from_dev, lt, it
import paper_2105_10375_b200 as dcp

d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
C, M, n_id = 333, 50, 400
head = dcp.DCPHead(C, d, 0, 1, 0, n_local_max=64, m_local_max=64)
pool = oracle.Pool(C, d, oracle.BF16)
for b in range(9):
    G = synth.unit_rows(5, synth.S_PRE, b, 0, M, d); y = synth.uniform_labels(5, synth.S_PRE_LAB, b, 0, M, n_id)
    head.enqueue(to_dev(G, 0), lt(y)); pool.enqueue(G, y)
torch.cuda.synchronize(); print("enqueue ok", flush=True)
X = synth.unit_rows(6, synth.S_INST, 0, 0, 30, d); y = synth.uniform_labels(6, synth.S_INST_LAB, 0, 0, 30, n_id)
t = time.time()
loss, dx = head.loss_fwd_bwd(to_dev(X, 0), lt(y), None, 64.0, 0.35)
torch.cuda.synchronize(); print("loss call ok", time.time() - t, flush=True)
try:
    head.check()
except Exception as e:
    print("check:", e)
ref = pool.loss(X, y, None, 64.0, 0.35)
st = head.row_stats(30)
print("N_pos gpu", st["N_pos"], "ref", ref.N_pos, "C_occ", st["C_occ"])
print("loss gpu", loss.item(), "ref", ref.L, ref.L_ce, ref.L_cos)
pos = ref.tslot >= 0
print("lse gpu", st["lse"][pos][:5], "ref", ref.lse[pos][:5])
print("ell gpu", st["ell"][pos][:5], "ref", ref.ell[pos][:5])
print("phi gpu", st["phi"][~pos][:5], "ref", ref.phi[~pos][:5])
g = from_dev(dx)
print("dx maxerr", np.abs(g - ref.dx).max(), "max", np.abs(ref.dx).max())
print("dx pos maxerr", np.abs(g[pos] - ref.dx[pos]).max(), "neg maxerr", np.abs(g[~pos] - ref.dx[~pos]).max(), np.abs(ref.dx[~pos]).max())
