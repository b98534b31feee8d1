"""World-size-2 CPU tests (gloo) of the multi-rank protocol.

Each process holds one slot shard of the pool and computes, in fp64 numpy, exactly the
per-shard partials the CUDA path exchanges: the C2 MAX all-reduce of (target write index,
norm bound), the C3 all-gather of per-row (l_rest, max, target exponent, phi), the owner-only
target term and the C4 sum of linear dx shares.  The merged result must equal the
single-pool oracle (D16).  This pins the merge rules with real collectives, on CPU."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _build_pool(C, d, seed):
    import oracle
    rng = np.random.default_rng(seed)
    pool = oracle.Pool(C, d, oracle.F32)
    for b in range(5):
        G = rng.standard_normal((37, d)).astype(np.float32)
        G /= np.linalg.norm(G, axis=1, keepdims=True)
        pool.enqueue(G, rng.integers(0, 60, 37))
    return pool


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    C, d, s, m = 150, 16, 30.0, 0.35
    pool = _build_pool(C, d, 7)
    rng = np.random.default_rng(11)
    N = 24
    X = rng.standard_normal((N, d)).astype(np.float32) * 2
    y = np.concatenate([pool.lab[rng.integers(0, pool.C_occ, 16)], 1000 + np.arange(8)])
    E = int(pool.E[0])
    C_occ = pool.C_occ
    lo, hi = C * rank // world, C * (rank + 1) // world
    T = pool.T.astype(np.float64)
    lab = pool.lab
    Xd = X.astype(np.float64)
    nrm = np.linalg.norm(Xd, axis=1)
    xh = Xd / nrm[:, None]
    occ = [c for c in range(lo, hi) if c < C_occ]
    # ---- C2: newest write index per row and the norm bound, MAX over ranks
    seq = lambda c: c + C * ((E - 1 - c) // C)  # noqa: E731
    tseq = np.full(N + 1, -1, dtype=np.int64)
    for i in range(N):
        hits = [seq(c) for c in occ if lab[c] == y[i]]
        tseq[i] = max(hits) if hits else -1
    tseq[N] = int(np.float64(max([np.linalg.norm(T[c]) for c in occ] + [0.0])).view(np.int64))
    t = torch.from_numpy(tseq)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tseq = t.numpy()
    tmax = np.int64(tseq[N]).view(np.float64)
    tslot = np.where(tseq[:N] >= 0, tseq[:N] % C, -1)
    pos = tslot >= 0
    N_pos, N_neg = int(pos.sum()), int((~pos).sum())
    b = s * tmax * (1 + 2 ** -10)                     # reference (natural-log units here)
    # ---- local partials over this shard
    scal = np.zeros((N, 4))
    O = np.zeros((N, d))
    mu = T[occ].sum(axis=0) if occ else np.zeros(d)
    for i in range(N):
        if pos[i]:
            e = {c: s * (xh[i] @ T[c]) - b for c in occ}
            tt = -np.inf
            if lo <= tslot[i] < hi:
                tt = e.pop(int(tslot[i])) - s * m
            vals = np.array(list(e.values())) if e else np.zeros(0)
            p = np.exp(vals)
            scal[i] = (p.sum(), vals.max() if len(vals) else -np.inf, tt, 0.0)
            O[i] = sum((np.exp(e[c]) * T[c] for c in e), np.zeros(d))
        else:
            scal[i] = (xh[i] @ mu / C_occ, 0, 0, 0)
    # ---- C3: all-gather the partials, finalise identically (rank order)
    gathered = [torch.zeros(N, 4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(scal))
    S = np.stack([g.numpy() for g in gathered])       # [W, N, 4]
    dxp = np.zeros((N, d))
    loss_terms = np.zeros(N)
    for i in range(N):
        if pos[i]:
            lr = S[:, i, 0].sum()
            tt = S[:, i, 2].max()
            l = lr + np.exp(tt)
            loss_terms[i] = np.log1p(lr * np.exp(-tt))
            owner = lo <= tslot[i] < hi
            g = (s / N_pos) * (O[i] / l - (lr / l) * T[tslot[i]] * owner)
        else:
            loss_terms[i] = S[:, i, 0].sum()
            g = mu / (N_neg * C_occ)
        dxp[i] = (g - (g @ xh[i]) * xh[i]) / nrm[i]
    L = loss_terms[pos].sum() / max(N_pos, 1) + loss_terms[~pos].sum() / max(N_neg, 1)
    # ---- C4: sum of the linear dx shares (all-reduce stands in for the reduce-scatter)
    t = torch.from_numpy(dxp)
    dist.all_reduce(t)
    dx = t.numpy()
    if rank == 0:
        ref = pool.loss(X, y, None, s, m)
        np.savez(out_path, L=L, ref_L=ref.L, dx=dx, ref_dx=ref.dx, tslot=tslot, ref_t=ref.tslot)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_protocol_equals_single_pool():
    out = os.path.join(tempfile.mkdtemp(), "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    np.testing.assert_array_equal(r["tslot"], r["ref_t"])
    assert abs(float(r["L"]) - float(r["ref_L"])) <= 1e-9 * abs(float(r["ref_L"]))
    np.testing.assert_allclose(r["dx"], r["ref_dx"], rtol=1e-8, atol=1e-11)


def _bench_max_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the bench's timing rule: every rank times its own loop, the job time is the MAX
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # shard plan used by the library: rank r owns [floor(r C/W), floor((r+1) C/W))
    C = 4_194_304 + 3
    lo, hi = C * rank // world, C * (rank + 1) // world
    spans = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(spans, torch.tensor([lo, hi]))
    if rank == 0:
        np.savez(out_path, t=t.numpy(), spans=np.stack([s.numpy() for s in spans]), C=C)
    dist.destroy_process_group()


def test_two_rank_timing_and_shard_plan():
    out = os.path.join(tempfile.mkdtemp(), "res.npz")
    mp.spawn(_bench_max_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    assert float(r["t"][0]) == 11.0
    sp = r["spans"]
    assert sp[0, 0] == 0 and sp[-1, 1] == int(r["C"]) and sp[0, 1] == sp[1, 0]
