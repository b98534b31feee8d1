"""Small parity check of one fused-kernel choice (F2C_KERNEL=pc4 / pc) against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
import synth  # noqa: E402
from helpers import from_dev, lt, to_dev  # noqa: E402
import paper_2105_10375_b200 as dcp  # noqa: E402

C, d, M, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
s = float(sys.argv[5]) if len(sys.argv) > 5 else 64.0
dcp.load_library()
head = dcp.DCPHead(C, d, dcp.BF16, world=1, rank=0, n_local_max=N, m_local_max=M)
pool = oracle.Pool(C, d, oracle.BF16)
rng = np.random.default_rng(5)
for b in range(C // M + 1):
    G = synth.unit_rows(5, synth.S_PRE, b, 0, M, d)
    y = rng.choice(20 * C, size=M, replace=False).astype(np.int64)
    head.enqueue(to_dev(G, synth.BF16), lt(y))
    pool.enqueue(G, y)
X = synth.unit_rows(6, synth.S_INST, 0, 0, N, d)
y = rng.integers(0, 20 * C, N).astype(np.int64)
y[: (3 * N) // 4] = pool.lab[rng.integers(0, pool.C_occ, (3 * N) // 4)]
loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, s, 0.35)
torch.cuda.synchronize()
head.check()
ref = pool.loss(X, y, None, s, 0.35)
g = from_dev(dx)
err = np.abs(g - ref.dx).max() / np.abs(ref.dx).max()
print(f"C={C} d={d} N={N} kernel={os.environ.get('F2C_KERNEL', 'auto')}: loss {float(loss.item()):.6f} "
      f"oracle {ref.L:.6f} rel {abs(float(loss.item()) - ref.L) / abs(ref.L):.2e}; dx max err / max|dx| {err:.2e}")
