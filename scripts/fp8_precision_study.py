"""NEXT-4 feasibility: can an fp8 (e4m3) pool meet BASELINE.json's parity bar?

A plain fp64 model of the DCP loss on a c2-like row set (d = 512, unit rows, pair noise
sigma = 0.3, s = 64, m = 0.35), with the operands of each GEMM rounded the way an fp8
`tcgen05.mma.kind::f8f6f4` path would round them (x_hat and T to e4m3 with a per-tensor
scale; P to e4m3 with a 2^8 scale), against the same model with bf16 operands (what the
shipped kernel does).  The bar is BJ:5: loss rel. error <= 2e-3, max|dx err| <= 1e-2 max|dx|.

usage: python scripts/fp8_precision_study.py [C] [N]
"""
import sys

import numpy as np
import torch

C = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
d, s, m = 512, 64.0, 0.35
rng = np.random.default_rng(0)
T = rng.standard_normal((C, d))
T /= np.linalg.norm(T, axis=1, keepdims=True)
tgt = rng.integers(0, C, N)
X = T[tgt] + 0.3 * rng.standard_normal((N, d))
X /= np.linalg.norm(X, axis=1, keepdims=True)


def q8(a, scale):
    t = torch.tensor(a * scale, dtype=torch.float32).to(torch.float8_e4m3fn).to(torch.float64).numpy()
    return t / scale


def qb(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()


def model(Xg1, Tg1, Tg2, qP):
    """loss and dL/dx_hat with GEMM-1 operands (Xg1, Tg1), GEMM-2 operand Tg2 and P rounding qP"""
    z = s * (Xg1 @ Tg1.T)
    z[np.arange(N), tgt] -= s * m
    mx = z.max(1, keepdims=True)
    p = np.exp(z - mx)
    l = p.sum(1, keepdims=True)
    ell = (mx[:, 0] + np.log(l[:, 0])) - z[np.arange(N), tgt]
    P = qP(p / l)
    G = P.copy()
    G[np.arange(N), tgt] -= 1.0
    return ell.mean(), s * (G @ Tg2) / N


ident = lambda a: a  # noqa: E731
L0, d0 = model(X, T, T, ident)
cases = {
    "bf16 operands (shipped kernel)": model(qb(X), qb(T), qb(T), qb),
    "fp8 GEMM 1 only (logits), bf16 GEMM 2": model(q8(X, 16), q8(T, 16), qb(T), qb),
    "bf16 GEMM 1, fp8 GEMM 2 (P and pool)": model(qb(X), qb(T), q8(T, 16), lambda a: q8(a, 256)),
    "fp8 everywhere (e4m3 pool, x_hat, P)": model(q8(X, 16), q8(T, 16), q8(T, 16), lambda a: q8(a, 256)),
}
print(f"C={C} N={N} d={d}: reference loss {L0:.4f}; bar: loss rel <= 2e-3, dx frac <= 1e-2")
for k, (L, dd) in cases.items():
    lr = abs(L - L0) / abs(L0)
    fr = np.abs(dd - d0).max() / np.abs(d0).max()
    ok = "PASS" if lr <= 2e-3 and fr <= 1e-2 else "FAIL"
    print(f"  {k:<42} loss rel {lr:.2e}   dx frac {fr:.3e}   {ok}")
