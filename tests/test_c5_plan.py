"""C5 (SURVEY 8(e) stage 0): the pure Eq. 7 enqueue routed to the owner ranks.  The plan is a host
function of the library (f2c_c5_plan, include/f2c_dcp.h), so it is checked here without a GPU:
against the definition (block row j -> slot (E + j) mod C, D6; slot p owned by the rank
whose range [floor(qC/W), floor((q+1)C/W)) holds it), and through real point-to-point collectives
(gloo, world 2 and 3, the same send / receive order the library issues to NCCL): every rank ends
with exactly the block rows it owns and receives only those bytes."""
import ctypes
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


@pytest.fixture(scope="module")
def lib():
    from paper_2105_10375_b200 import build
    build.build()
    import paper_2105_10375_b200 as m
    L = m.load_library()
    L.f2c_c5_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_int64]
    L.f2c_c5_plan.restype = ctypes.c_int64
    return L


def plan(L, C, W, E, m):
    buf = np.zeros((2 * W + 2, 4), dtype=np.int64)
    n = L.f2c_c5_plan(C, W, E, m, buf.ctypes.data_as(ctypes.c_void_p), len(buf))
    assert n >= 0
    return buf[:n]


def owner(p, C, W):
    return next(q for q in range(W) if C * q // W <= p < C * (q + 1) // W)


@pytest.mark.parametrize("C,W,m", [(100, 2, 10), (101, 3, 33), (4097, 8, 512), (64, 8, 8), (1000, 7, 1)])
def test_plan_matches_definition(lib, C, W, m):
    rng = np.random.default_rng(C + W)
    for E in list(range(0, 3 * C, max(1, C // 7))) + list(rng.integers(0, 10**9, 20)):
        P = plan(lib, C, W, int(E), m)
        assert len(P) <= 2 * W + 1
        seen = np.zeros(W * m, dtype=int)
        prev = (-1, -1)
        for src, dst, j, n in P:
            assert n >= 1 and src * m <= j and j + n <= (src + 1) * m          # rows of one sender
            assert (src, j) > prev                                             # issue order
            prev = (src, j)
            slots = (E + j + np.arange(n)) % C
            assert np.all(np.diff(slots) == 1)                                 # contiguous in the shard
            assert all(owner(int(p), C, W) == dst for p in slots)              # the owner receives
            seen[j:j + n] += 1
        assert np.all(seen == 1)                                               # every row exactly once


def test_plan_rejects_bad_arguments(lib):
    buf = np.zeros((4, 4), dtype=np.int64)
    P = buf.ctypes.data_as(ctypes.c_void_p)
    assert lib.f2c_c5_plan(10, 2, 0, 6, P, 4) == -1        # W m > C
    assert lib.f2c_c5_plan(100, 8, 0, 10, P, 1) == -1      # too few piece slots
    assert lib.f2c_c5_plan(100, 2, -1, 10, P, 4) == -1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path, C, m, E_list):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2105_10375_b200 as pkg
    L = pkg.load_library()
    L.f2c_c5_plan.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_int64]
    L.f2c_c5_plan.restype = ctypes.c_int64
    d = 6
    ok = True
    lo, hi = C * rank // world, C * (rank + 1) // world
    for E in E_list:
        # this rank's block rows (global rows rank*m ..): features encode (row, column)
        rows = rank * m + np.arange(m)
        g = torch.tensor(rows[:, None] * 100 + np.arange(d)[None, :], dtype=torch.float32)
        y = torch.tensor(rows * 7 + 3, dtype=torch.int64)
        stage_g = torch.full((world * m, d), -1.0)
        stage_y = torch.full((world * m,), -1, dtype=torch.int64)
        P = plan(L, C, world, E, m)
        recv_bytes = 0
        ops, landed = [], []
        for src, dst, j, n in P:          # the library's issue order
            src, dst, j, n = int(src), int(dst), int(j), int(n)
            if src == dst == rank:
                stage_g[j:j + n] = g[j - rank * m:j - rank * m + n]
                stage_y[j:j + n] = y[j - rank * m:j - rank * m + n]
            elif src == rank:
                ops.append(dist.P2POp(dist.isend, g[j - rank * m:j - rank * m + n].contiguous(), dst))
                ops.append(dist.P2POp(dist.isend, y[j - rank * m:j - rank * m + n].contiguous(), dst))
            elif dst == rank:
                bg = torch.empty((n, d))
                by = torch.empty((n,), dtype=torch.int64)
                ops.append(dist.P2POp(dist.irecv, bg, src))
                ops.append(dist.P2POp(dist.irecv, by, src))
                recv_bytes += n * d * 4
                landed.append((j, n, bg, by))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        for r in reqs:
            r.wait()
        for j, n, bg, by in landed:
            stage_g[j:j + n] = bg
            stage_y[j:j + n] = by
        # rows whose slot this rank owns are all present, correct, and nothing else arrived
        own = [j for j in range(world * m) if lo <= (E + j) % C < hi]
        for j in own:
            ok &= bool(torch.equal(stage_g[j], torch.tensor(j * 100 + np.arange(d), dtype=torch.float32)))
            ok &= int(stage_y[j]) == j * 7 + 3
        own_remote = [j for j in own if j // m != rank]
        ok &= recv_bytes == len(own_remote) * d * 4
    dist.barrier()
    dist.destroy_process_group()
    with open(out_path + f".{rank}", "w") as f:
        f.write("ok" if ok else "bad")


@pytest.mark.parametrize("world,C,m", [(2, 50, 9), (3, 61, 13)])
def test_c5_routing_with_gloo(lib, world, C, m):
    port = _free_port()
    out = tempfile.mktemp()
    E_list = [0, 5, C - 3, C + 11, 3 * C - 1, 12345]
    mp.spawn(_worker, args=(world, port, out, C, m, E_list), nprocs=world, join=True)
    for r in range(world):
        assert open(out + f".{r}").read() == "ok"
