#!/usr/bin/env python
"""Benchmark of the F2C DCP head on B200 (contract: DESIGN.md section 8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c1]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)
  python bench.py --impl reference ...                   (the CPU oracle arm)

One step = one pass of the whole hot path: enqueue of the
step's G-Net identity block, the fused loss forward+backward over the mixed P-Net
batch, and the G-Net EMA over a 65M-parameter fp32 vector.  Rank 0 prints ONE JSON
line.  Inputs: synthetic and seeded (synth/), pool prefilled through the enqueue
kernel (D20).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "DCP head fwd+bwd+enqueue samples/s"
UNIT = "samples/s"
EMA_PARAMS = 65_000_000


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "_fallback": True}


# --------------------------------------------------------------------------- CPU oracle timing
def oracle_sample_time(cfg: synth.Config, world: int, C_sample: int, k_rows: int, step: int = 0):
    """Time the (unmodified) oracle on a bounded sample of workload `cfg`: a sub-pool of
    C_sample slots (tiled seeded rows + the step's identity block) and k_rows sampled
    batch rows (half identity rows, half instance rows).  Both parts of the oracle are
    linear in the pool size, so the full step time is extrapolated by C / C_sample."""
    import oracle
    d = cfg.d
    stp_parts = [synth.step_inputs(cfg, step, r, world) for r in range(world)]
    x = np.concatenate([s.x for s in stp_parts])
    y = np.concatenate([s.y for s in stp_parts])
    g = np.concatenate([s.g for s in stp_parts])
    gy = np.concatenate([s.gy for s in stp_parts])
    N, M = len(y), len(gy)
    pool = oracle.Pool(C_sample, d, oracle.BF16)
    blk = 4096
    base = synth.unit_rows(cfg.seed, synth.S_PRE, 0, 0, blk, d, synth.BF16)
    fill = C_sample - M
    for o in range(0, fill, blk):
        n = min(blk, fill - o)
        pool.enqueue(base[:n], synth.uniform_labels(cfg.seed, synth.S_PRE_LAB, 0, o, n, cfg.n_id))
    pool.enqueue(g, gy)
    t0 = time.perf_counter()
    pool.loss_rows(x, y, None, cfg.s, cfg.m, np.zeros(0, np.int64))
    t_prep = time.perf_counter() - t0
    half = max(1, k_rows // 2)
    # identity rows of rank 0 sit at [M_loc, 2 M_loc); instance rows at [0, M_loc)
    rows = np.concatenate([np.arange(half), cfg.M_loc + np.arange(half)])[:k_rows]
    t0 = time.perf_counter()
    res = pool.loss_rows(x, y, None, cfg.s, cfg.m, rows)
    t_rows = time.perf_counter() - t0 - t_prep
    scale = cfg.C / C_sample
    t_step = (t_prep + N * max(t_rows, 1e-9) / len(rows)) * scale
    return dict(t_step=t_step, t_prep=t_prep, t_rows=t_rows, rows=len(rows), N=N, N_pos=res["N_pos"],
                wall=t_prep + t_rows)


def cpu_baseline(cfg, world, budget_s=20.0):
    C_s = min(cfg.C, 131072)
    k = 16
    r = oracle_sample_time(cfg, world, C_s, k)
    if r["wall"] < budget_s / 3 and C_s < cfg.C:  # grow the sample toward ~budget
        k = int(min(128, k * max(1.0, budget_s / max(r["wall"], 1e-3) / 2)))
        r = oracle_sample_time(cfg, world, C_s, k)
    return dict(value=r["N"] / r["t_step"], unit=UNIT, cores=1, kind="oracle",
                sample=(f"fp64 C oracle (1 thread) on {r['rows']} sampled rows (half identity, half "
                        f"instance) of step 0 against a {C_s}-slot sub-pool, plus the full "
                        f"target-resolve/mu pass over that sub-pool; step time extrapolated x"
                        f"{cfg.C / C_s:.1f} to C={cfg.C} and to all {r['N']} rows"),
                sample_wall_s=round(r["wall"], 2))


def run_reference(args, cfg, world):
    """--impl reference: the oracle as it stands, timed on the host cores, one bounded
    sample per step (the CPU arm of this tier)."""
    K, W = args.steps, args.warmup
    budget = max(0.5, 150.0 / max(1, K + W))           # seconds of oracle work per step
    C_s = min(cfg.C, 16384)
    probe = oracle_sample_time(cfg, world, C_s, 2)
    per_row = max(probe["t_rows"] / 2, 1e-6)
    C_s = int(min(cfg.C, max(4096, C_s * budget / max(probe["wall"], 1e-3) / 2)))
    C_s = max(4096, min(C_s, cfg.C, 262144))
    times = []
    for i in range(W + K):
        r = oracle_sample_time(cfg, world, C_s, 2, step=i % 4)
        if i >= W:
            times.append(r["t_step"])
    N = probe["N"]
    tot = sum(times)
    val = K * N / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * tot / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(cfg, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"per step: 2 sampled rows against a {C_s}-slot sub-pool + "
                                       f"the resolve/mu pass, extrapolated x{cfg.C / C_s:.1f} to "
                                       f"C={cfg.C} and to {N} rows; per-row cost {per_row:.3f}s"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _variant(args):
    v = []
    if args.lcos:
        v.append(f"lcos={args.lcos}")
    if args.excl_dup:
        v.append("exclude-stale-duplicates")
    if args.refresh:
        v.append("refresh-in-place enqueue")
    return ", ".join(v) if v else "default (D8, D10, pure Eq. 7)"


def _config(cfg, world, ema_overlap=True, K=1, variant="default (D8, D10, pure Eq. 7)"):
    return {"workload": cfg.name, "model": "DCP head (F2C)", "C": cfg.C, "C_per_gpu": cfg.C // world,
            "d": cfg.d, "global_batch": cfg.N_loc() * world, "M_glob": cfg.M_glob(world),
            "n_id": cfg.n_id, "s": cfg.s, "m": cfg.m, "pair_noise_sigma": cfg.sigma,
            "ema_params": EMA_PARAMS, "K": K, "variant": variant, "parallelism": f"slot-range sharded pool x{world}",
            "l2_hygiene": "inputs larger than L2 (the pool streams through L2 every step)",
            "prefill": "normalised Gaussian rows + uniform labels through the enqueue kernel (D20)",
            "ema_stream": ("low-priority side stream, after the step's loss (overlaps the next step's "
                           "head kernels; joined before the timed region ends)") if ema_overlap else "same stream"}


# --------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200", "-i",
                                       str(gpu_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [ln.strip().split(",") for ln in open(self.f.name) if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- GPU arm
def run_ours(args, cfg, world, rank, local_rank, device_only=False):
    import torch
    import torch.distributed as dist
    import paper_2105_10375_b200 as dcp

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    M, N_loc, d = cfg.M_loc, cfg.N_loc(), cfg.d
    uid = None
    if world > 1:
        # the library's NCCL communicator is bootstrapped from a unique id made by rank 0
        # and broadcast over the torch process group (torch only for plumbing)
        if rank == 0:
            raw = bytes(torch.cuda.nccl.unique_id())
            t = torch.tensor(list(raw), dtype=torch.uint8, device=dev)
        else:
            t = torch.zeros(128, dtype=torch.uint8, device=dev)
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().tolist())
    K = args.K
    head = dcp.DCPHead(cfg.C, d, dcp.BF16, world, rank if world > 1 else 0, n_local_max=N_loc,
                       m_local_max=M, nccl_uid=uid, device=dev, K=K)
    if args.lcos:  # NEXT-3 variants (timing of the variant paths)
        mode, hinge, lam = args.lcos.split(",")
        head.set_lcos(int(mode), bool(int(hinge)), float(lam))
    if args.excl_dup:
        head.set_dup_mode(True)
    # the head runs on a high-priority stream; the G-Net EMA (a10, independent of the head's
    # data) on a low-priority side stream, after the step's loss, so that it overlaps the
    # head's latency-bound kernels of the next step instead of extending the step
    stream = torch.cuda.Stream(device=dev, priority=-1)
    side = torch.cuda.Stream(device=dev, priority=0)
    torch.cuda.set_stream(stream)
    ev_loss = torch.cuda.Event()

    # ---- prefill (D20): seeded GPU RNG, normalised rows, uniform labels, through K1
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg.seed * 1000 + rank)
    nblk = cfg.prefill_blocks(world)
    for b in range(nblk):
        gb = torch.randn(M, K, d, device=dev, generator=gen) if K > 1 else torch.randn(M, d, device=dev, generator=gen)
        gb = (gb / gb.norm(dim=-1, keepdim=True)).to(torch.bfloat16)
        yb = torch.randint(0, cfg.n_id, (M,), device=dev, generator=gen)
        head.enqueue(gb, yb)
    torch.cuda.synchronize()
    if args.refresh:  # NEXT-3: refresh-in-place enqueue for the timed steps
        head.set_enqueue_mode(True)

    # ---- per-step inputs: a ring of R seeded steps (synth), pinned host + device copies
    R = args.ring
    host, devin = [], []
    for t in range(R):
        s = synth.step_inputs(cfg, t, rank, world)
        hx = torch.from_numpy(s.x.view(np.int16)).view(torch.bfloat16).pin_memory()
        g = s.g
        if K > 1:  # K features per identity (NEXT-1): the G-Net pair plus K-1 more noisy copies
            g = np.stack([s.g] + [synth.pair_rows(cfg.seed, 1_000_000 * k + t, rank * M, M, d, cfg.sigma)[1]
                                  for k in range(1, K)], axis=1)
        hg = torch.from_numpy(np.ascontiguousarray(g).view(np.int16)).view(torch.bfloat16).pin_memory()
        hy = torch.from_numpy(s.y).pin_memory()
        hp = torch.from_numpy(s.pairing).pin_memory()
        hgy = torch.from_numpy(s.gy).pin_memory()
        host.append((hx, hy, hp, hg, hgy))
        devin.append(tuple(a.to(dev) for a in (hx, hy, hp, hg, hgy)))
    h2d_bytes = sum(a.numel() * a.element_size() for a in host[0])
    # G-Net / P-Net parameter vectors for the EMA (a10), resident on the device
    ema_p = torch.randn(EMA_PARAMS, device=dev, generator=gen) * 0.05
    ema_g = torch.randn(EMA_PARAMS, device=dev, generator=gen) * 0.05
    dx = torch.empty(N_loc, d, dtype=torch.bfloat16, device=dev)
    loss = torch.zeros((), dtype=torch.float32, device=dev)
    launches = [0]

    def step(inp):
        x, y, pr, g, gy = inp
        head.enqueue(g, gy)                                  # a1 (D4: enqueue first)
        launches[0] += head.last_launch_count()
        head.loss_fwd_bwd(x, y, pr, cfg.s, cfg.m, dx=dx, loss=loss)  # a2-a9
        launches[0] += head.last_launch_count()
        if args.ema_overlap:
            ev_loss.record(stream)
            side.wait_event(ev_loss)
            dcp.gnet_ema(ema_p, ema_g, 0.999, stream=side)   # a10
        else:
            dcp.gnet_ema(ema_p, ema_g, 0.999)
        launches[0] += head.last_launch_count()

    def join():  # the timed region ends after the side stream's last EMA
        stream.wait_stream(side)

    for i in range(args.warmup):
        step(devin[i % R])
    join()
    timing_experiment = bool(os.environ.get("F2C_DBG_FLAGS"))  # kernel parts disabled: results void
    if not timing_experiment:
        head.check()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxrank(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed run (value)
    K = args.steps
    barrier()
    clk = Clocks(local_rank) if rank == 0 else None
    head.profile(True)
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    torch.cuda.nvtx.range_push("timed_steps")  # ncu --nvtx-include timed_steps/ selects these launches
    for i in range(K):
        step(devin[i % R])
    join()
    torch.cuda.nvtx.range_pop()
    e1.record(stream)
    barrier()
    clocks = clk.stop() if clk else None
    ms = maxrank(e0.elapsed_time(e1))
    n_launch = launches[0]
    main_ms, main_n, npos_sum = head.profile_read()
    head.profile(False)
    if not timing_experiment:
        head.check()
    value = K * N_loc * world / (ms / 1e3)

    if device_only:
        if rank != 0:
            return None
        pk = _peaks()
        C_loc = cfg.C // world
        npos_avg = npos_sum / max(1, main_n)
        t_launch = main_ms / max(1, main_n) / 1e3
        achieved = 4.0 * npos_avg * C_loc * d / t_launch / 1e12
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        head.close()
        return {"workload": cfg.name, "value": value, "unit": UNIT, "ms_per_step": ms / K,
                "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak, "avg_launch_ms": t_launch * 1e3, "N_pos_avg": npos_avg},
                "clocks": clocks, "config": _config(cfg, world, args.ema_overlap, args.K, _variant(args))}

    # ---- end-to-end through the public API with host buffers (e2e): every step copies its
    # inputs from pinned host memory and reads the loss back.  The copies run on a copy
    # stream into double-buffered device inputs, so step i+1's upload overlaps step i.
    loss_host = torch.zeros((), dtype=torch.float32).pin_memory()
    bufs = [tuple(torch.empty_like(a) for a in devin[0]) for _ in range(2)]
    copy_st = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    copy_st.wait_event(e2)                       # no upload before the timed region starts
    for i in range(K):
        b = i % 2
        if i >= 2:
            copy_st.wait_event(freed[b])         # step i-2 is done with buffer b
        with torch.cuda.stream(copy_st):
            for dst, src in zip(bufs[b], host[i % R]):
                dst.copy_(src, non_blocking=True)
        copied[b].record(copy_st)
        stream.wait_event(copied[b])
        step(bufs[b])
        freed[b].record(stream)
        loss_host.copy_(loss, non_blocking=True)
    join()
    stream.wait_stream(copy_st)
    e3.record(stream)
    barrier()
    ms_e2e = maxrank(e2.elapsed_time(e3))
    value_e2e = K * N_loc * world / (ms_e2e / 1e3)

    if rank != 0:
        head.close()
        return None
    pk = _peaks()
    C_loc = cfg.C // world
    npos_avg = npos_sum / max(1, main_n)
    flops_alg = 4.0 * npos_avg * C_loc * d          # GEMM 1 + GEMM 2 on the in-pool rows
    t_launch = main_ms / max(1, main_n) / 1e3
    achieved = flops_alg / t_launch / 1e12
    peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    # MMA rows: 128-row groups (TMEM lanes); a last group of <= 64 rows runs with M = 64
    # (dcp_pc_kernel's tail unit; evaluated at the average N_pos)
    tail = npos_avg - math.floor(npos_avg / 128) * 128
    rows_exec = math.floor(npos_avg / 128) * 128 + (0 if tail == 0 else 64 if tail <= 64 else 128)
    flops_exec = 4.0 * rows_exec * C_loc * d
    traffic = None
    prof_file = os.path.join(ROOT, "profiles", f"ncu_main_{cfg.name}.json")
    if os.path.exists(prof_file):
        try:
            traffic = json.load(open(prof_file)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": _config(cfg, world, args.ema_overlap, args.K, _variant(args)),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "dcp_pc_kernel (producer: TMEM-A logits GEMM + softmax -> DSMEM P; consumer: P x pool GEMM, O in TMEM)",
                     "algorithmic_flops_per_launch": flops_alg,
                     "executed_mma_flops_per_launch": flops_exec,
                     "tensor_pipe_frac": flops_exec / t_launch / 1e12 / peak,
                     "avg_launch_ms": t_launch * 1e3, "N_pos_avg": npos_avg,
                     "peak_kind": "measured sustained bf16 (MEASURED_PEAKS.json), kernel timed inside a long step",
                     "main_kernel_share_of_step": main_ms / ms},
        "e2e": {"value": value_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": 4, "ms_per_step": ms_e2e / K},
        "gpu_launches": n_launch,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, world)
    return line


def kernel_bench(args):
    """HBM-bound kernels in isolation (SURVEY 8(d) 'enqueue and EMA evidence'): the
    enqueue of a 262,144-row bf16 block (256 MB in, 256 MB out) into a 4M-slot pool, and
    the G-Net EMA over 65M fp32 parameters (780 MB).  CUDA events, best of 10 after warm-up."""
    import torch
    import paper_2105_10375_b200 as dcp
    pk = _peaks()
    dev = torch.device("cuda", 0)
    out = {}
    M, C, d = 262_144, 4_194_304, 512
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=8, m_local_max=M, device=dev)
    g = torch.randn(M, d, device=dev).bfloat16()
    y = torch.arange(M, device=dev, dtype=torch.int64)
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        head.enqueue(g, y)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    byt = M * d * 2 * 2 + M * 8 * 2
    out["enqueue"] = {"rows": M, "bytes": byt, "best_ms": min(ts), "GBps": byt / (min(ts) * 1e-3) / 1e9,
                      "frac_of_measured_copy": byt / (min(ts) * 1e-3) / 1e9 / pk["hbm_gbs"]}
    del head
    p = torch.randn(EMA_PARAMS, device=dev) * 0.05
    gq = torch.randn(EMA_PARAMS, device=dev) * 0.05
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dcp.gnet_ema(p, gq, 0.999)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    byt = EMA_PARAMS * 4 * 3
    out["ema"] = {"params": EMA_PARAMS, "bytes": byt, "best_ms": min(ts), "GBps": byt / (min(ts) * 1e-3) / 1e9,
                  "frac_of_measured_copy": byt / (min(ts) * 1e-3) / 1e9 / pk["hbm_gbs"]}
    print(json.dumps({"kernel_bench": out, "peak_hbm_GBps": pk["hbm_gbs"]}), flush=True)


def c4_rank_config(frac, n_glob):
    """One rank of the W=8 c4 point (C = frac * 10M, global batch n_glob) as a 1-GPU workload."""
    base = synth.c4_point(frac, n_glob, world=8)
    return synth.scaled(base, name=f"c4r_{int(round(frac * 100))}_{n_glob}", C=base.C // 8,
                        M_loc=n_glob // 2, n_id=base.n_id // 8)


def _workload(name):
    if name.startswith("c4r_"):  # c4r_<pct>_<global batch>: one rank of a W=8 c4 point
        _, pct, n = name.split("_")
        return c4_rank_config(int(pct) / 100, int(n))
    if name.startswith("c3r_"):  # c3r_<W>: the compute of one rank of c3 at W ranks (no collectives)
        W = int(name.split("_")[1])
        base = synth.CONFIGS["c3"]
        return synth.scaled(base, name=name, C=base.C // W, M_loc=base.M_loc * W, n_id=base.n_id // W)
    return synth.CONFIGS[name]


def sweep_c4(args):
    """BJ:11's pool-ratio x batch sweep, per-rank view on ONE GPU: for each point (C = 1/2/5/10 %
    of 10M ids, global batch N in {2048, 8192, 16384}) run the compute ONE rank of the W=8 job
    does -- all N global rows against its C/8-slot shard, plus the enqueue of the N/2-row global
    block and the 65M-parameter EMA -- device-resident (n_ID / 8 keeps the instance rows' in-pool
    rate C / n_ID of the sharded job).  Collectives (C1-C5) are excluded, so
    N / t_step is an upper bound of the W=8 job's samples/s; the driver's 8-GPU run measures the
    real thing.  Prints one JSON line (evidence for profiles/, not the bench contract line)."""
    import torch
    pts = []
    for frac in (0.01, 0.02, 0.05, 0.10):
        for n_glob in (2048, 8192, 16384):
            base = synth.c4_point(frac, n_glob, world=8)
            cfg = c4_rank_config(frac, n_glob)
            r = run_ours(args, cfg, 1, 0, 0, device_only=True)
            pts.append({"C_global": base.C, "C_per_rank": cfg.C, "global_batch": n_glob,
                        "ms_per_step": r["ms_per_step"], "upper_bound_w8_samples_per_s": r["value"],
                        "fused_kernel_ms": r["roofline"]["avg_launch_ms"],
                        "fused_kernel_frac": r["roofline"]["frac"], "N_pos_avg": r["roofline"]["N_pos_avg"],
                        "clocks": r["clocks"]})
            torch.cuda.empty_cache()
    print(json.dumps({"sweep": "c4 (BJ:11), one rank of W=8 on one B200, collectives excluded",
                      "steps": args.steps, "warmup": args.warmup, "points": pts}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3",
                    help="c1 | c2 | c3 | c4r_<pct>_<global batch> (one rank of a W=8 c4 point) | "
                         "c3r_<W> (one rank of c3 at W GPUs, collectives excluded)")
    ap.add_argument("--ring", type=int, default=8)
    ap.add_argument("--K", type=int, default=1, help="features per pool slot (NEXT-1; the paper's default is 2)")
    ap.add_argument("--lcos", default="", help="NEXT-3 L_cos variant 'phi_mode,hinge,lambda' (e.g. 2,0,1 = max)")
    ap.add_argument("--excl-dup", action="store_true", help="NEXT-3: exclude stale self-duplicates")
    ap.add_argument("--refresh", action="store_true", help="NEXT-3: refresh-in-place enqueue")
    ap.add_argument("--ema-overlap", type=int, default=1,
                    help="1: G-Net EMA on a low-priority side stream (overlaps the head's small kernels)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-bench", action="store_true", help="HBM-bound kernels alone (enqueue, EMA)")
    ap.add_argument("--sweep-c4", action="store_true", help="BJ:11 sweep, one rank of W=8 per point (evidence)")
    ap.add_argument("--also", default="c2", help="extra single-GPU workloads measured device-resident "
                    "(the north-star 1M-slot config c2 by default); 'none' to skip")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = _workload(args.workload)
    if args.kernel_bench:
        kernel_bench(args)
        return
    if args.sweep_c4:
        sweep_c4(args)
        return
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, cfg, world, rank, local_rank)
    extras = [w.strip("'\"") for w in args.also.split(",")]
    extras = [w for w in extras if w and w != "none" and w != args.workload] if world == 1 else []
    if extras:
        import torch
        torch.cuda.empty_cache()
        line["also"] = [run_ours(args, _workload(w), world, rank, local_rank, device_only=True)
                        for w in extras]
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
