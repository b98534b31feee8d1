#!/usr/bin/env python
"""Benchmark of the F2C DCP head on B200 (contract: DESIGN.md section 8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c1]
      --gpus N > 1 without WORLD_SIZE in the environment re-launches this script under
      torch.distributed.run with N ranks (one process per GPU, NCCL); under torchrun
      WORLD_SIZE must equal N.
  python bench.py --impl reference ...                   (the CPU oracle arm)

One step = one pass of the whole hot path: enqueue of the
step's G-Net identity block, the fused loss forward+backward over the mixed P-Net
batch, and the G-Net EMA over a 65M-parameter fp32 vector.  Rank 0 prints ONE JSON
line.  Before anything is timed, every rank runs a small W-rank step whose loss, dx and
pool state are checked against the fp64 oracle on the rank-ordered concatenation (D16,
pin P9): `w_parity` in the line; a failing check prints no value and exits 1.
Inputs: synthetic and seeded (synth/), pool prefilled through the enqueue kernel (D20).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
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
LOSS_RTOL, DX_FRAC = 2e-3, 1e-2   # BJ:5 parity bars (also tests/helpers.py)


def _peaks():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        pk["_source"] = "MEASURED_PEAKS.json (driver-measured on this pool's B200s)"
        return pk
    except Exception:
        # /opt/skills/guides/B200_PROFILING.md fallback figures
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "_source": "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"}


def host_cpu():
    """The host the CPU legs run on: lscpu model, nproc, governor."""
    model = platform.processor() or "?"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    gov = None
    try:
        gov = open("/sys/devices/system/cpu/cpu0/cpufreq/scaling_governor").read().strip()
    except Exception:
        gov = "n/a (no cpufreq in this guest)"
    try:
        affinity = len(os.sched_getaffinity(0))
    except Exception:
        affinity = os.cpu_count()
    return {"lscpu_model": model, "nproc": os.cpu_count(), "affinity_cpus": affinity, "governor": gov}


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
    extrap = cfg.C / C_s
    return dict(value=r["N"] / r["t_step"], unit=UNIT, cores=1, kind="oracle",
                sample=(f"fp64 C oracle (1 thread) on {r['rows']} sampled rows (half identity, half "
                        f"instance) of step 0 against a {C_s}-slot sub-pool, plus the full "
                        f"target-resolve/mu pass over that sub-pool; step time extrapolated x"
                        f"{extrap:.1f} to C={cfg.C} and to all {r['N']} rows"
                        + (" (an estimate, not a timing of the full step)" if extrap > 1 or r["rows"] < r["N"] else "")),
                sample_wall_s=round(r["wall"], 2), extrapolated=bool(extrap > 1 or r["rows"] < r["N"]),
                host=host_cpu())


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
    times, walls = [], []
    for i in range(W + K):
        r = oracle_sample_time(cfg, world, C_s, 2, step=i % 4)
        if i >= W:
            times.append(r["t_step"])
            walls.append(r["wall"])
    N = probe["N"]
    tot = sum(times)
    val = K * N / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * tot / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(cfg, world),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"per step: 2 sampled rows against a {C_s}-slot sub-pool + "
                                       f"the resolve/mu pass, extrapolated x{cfg.C / C_s:.1f} to "
                                       f"C={cfg.C} and to {N} rows (an estimate, not a timing of the "
                                       f"full step); per-row cost {per_row:.3f}s",
                             "sample_wall_s_per_step": round(sum(walls) / max(1, len(walls)), 3),
                             "extrapolated": True, "host": host_cpu()},
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
    return {"workload": cfg.name, "C": cfg.C, "C_per_gpu": cfg.C // world,
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
                                       "--format=csv,noheader,nounits", "-lms", "100", "-i",
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
        sm, mx, pw, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                pw.append(float(r[3]))
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "sm_mhz_min": min(sm), "power_w_max": max(pw) if pw else None}


# --------------------------------------------------------------------------- multi-rank plumbing
def _nccl_uid(world, rank, dev):
    """The library's NCCL communicator is bootstrapped from a unique id made by rank 0 and
    broadcast over the torch process group (torch only for plumbing)."""
    import paper_2105_10375_b200 as dcp
    return None if world == 1 else dcp.nccl_unique_id(dev)


def w_parity(world, rank, local_rank, dev, emulate=0):
    """Self-check before timing: one W-rank step (prefill, enqueue of the
    step's identity block, loss) of a small seeded workload with ragged shards and a wrapped
    ring, through the same NCCL protocol as the timed run; loss, dx and the pool state are
    gathered to rank 0 and compared with the fp64 oracle on the rank-ordered concatenation
    (D16, pin P9).  emulate > 1 (W = 1 only): the same check through the emulated world of
    `emulate` ranks on one device.  Returns the result dict on every rank (ok broadcast)."""
    import torch
    import torch.distributed as dist
    import paper_2105_10375_b200 as dcp
    Wl = world if world > 1 else max(1, emulate)
    cfg = synth.scaled(synth.CONFIGS["c1"], name="w_parity", C=1000 * Wl + 37, M_loc=32,
                       n_id=3000 * Wl, prefill=0, seed=synth.SEED_BASE + 77)
    M, N_loc, d = cfg.M_loc, cfg.N_loc(), cfg.d
    uid = _nccl_uid(world, rank, dev)
    if world > 1:
        head = dcp.DCPHead(cfg.C, d, dcp.BF16, world, rank, n_local_max=N_loc, m_local_max=M, nccl_uid=uid,
                           device=dev)
    else:
        head = dcp.DCPHead(cfg.C, d, dcp.BF16, Wl, -1 if Wl > 1 else 0, n_local_max=N_loc, m_local_max=M,
                           device=dev)
    my_ranks = [rank] if world > 1 else list(range(Wl))

    def block(parts):
        return np.concatenate(parts) if len(parts) > 1 else parts[0]

    nblk = cfg.prefill_blocks(Wl) + 3          # the ring wraps
    for b in range(nblk):
        parts = [synth.prefill_block(cfg, b, r, Wl) for r in my_ranks]
        g = block([p[0] for p in parts])
        y = block([p[1] for p in parts])
        head.enqueue(torch.from_numpy(g.view(np.int16)).view(torch.bfloat16).to(dev), torch.from_numpy(y).to(dev))
    st = [synth.step_inputs(cfg, 0, r, Wl) for r in my_ranks]
    head.enqueue(torch.from_numpy(block([s.g for s in st]).view(np.int16)).view(torch.bfloat16).to(dev),
                 torch.from_numpy(block([s.gy for s in st])).to(dev))
    x = torch.from_numpy(block([s.x for s in st]).view(np.int16)).view(torch.bfloat16).to(dev)
    loss, dx = head.loss_fwd_bwd(x, torch.from_numpy(block([s.y for s in st])).to(dev),
                                 torch.from_numpy(block([s.pairing for s in st])).to(dev), cfg.s, cfg.m)
    torch.cuda.synchronize()
    err = None
    try:
        head.check()
    except Exception as e:  # a latched device error fails the check below
        err = str(e)
    feats, labs, E = head.get_state()
    L = float(loss.item())
    dx_u16 = dx.view(torch.int16).cpu().numpy().view(np.uint16)
    head.close()
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (L, dx_u16, feats, labs, E, err))
    else:
        gathered = [(L, dx_u16, feats, labs, E, err)]
    res = None
    ok = 1
    if rank == 0:
        import oracle
        pool = oracle.Pool(cfg.C, d, oracle.BF16)
        for b in range(nblk):
            parts = [synth.prefill_block(cfg, b, r, Wl) for r in range(Wl)]
            pool.enqueue(np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))
        sa = [synth.step_inputs(cfg, 0, r, Wl) for r in range(Wl)]
        pool.enqueue(np.concatenate([s.g for s in sa]), np.concatenate([s.gy for s in sa]))
        ref = pool.loss(np.concatenate([s.x for s in sa]), np.concatenate([s.y for s in sa]),
                        np.concatenate([s.pairing for s in sa]), cfg.s, cfg.m)
        dxg = oracle.bf16_to_f64(np.concatenate([g[1] for g in gathered]))
        losses = [g[0] for g in gathered]
        feats_all = np.concatenate([g[2] for g in gathered])
        labs_all = np.concatenate([g[3] for g in gathered])
        loss_rel = abs(losses[0] - ref.L) / abs(ref.L)
        dx_frac = float(np.abs(dxg - ref.dx).max() / np.abs(ref.dx).max())
        pos = ref.tslot >= 0
        dx_frac_out = (float(np.abs(dxg[~pos] - ref.dx[~pos]).max() / np.abs(ref.dx[~pos]).max())
                       if (~pos).any() else 0.0)
        state_ok = (all(g[4] == int(pool.E[0]) for g in gathered) and np.array_equal(labs_all, pool.lab)
                    and np.array_equal(feats_all[: pool.C_occ], pool.T[: pool.C_occ]))
        same_loss = all(v == losses[0] for v in losses)
        errs = [g[5] for g in gathered if g[5]]
        ok = int(loss_rel <= LOSS_RTOL and dx_frac <= DX_FRAC and dx_frac_out <= DX_FRAC and state_ok
                 and same_loss and not errs)
        res = {"ok": bool(ok), "world": Wl, "transport": ("nccl" if world > 1 else
                                                          ("emulated" if Wl > 1 else "single")),
               "loss_rel": loss_rel, "dx_frac": dx_frac, "dx_frac_out_of_pool": dx_frac_out,
               "state_bitexact": bool(state_ok), "loss_identical_on_ranks": bool(same_loss),
               "device_errors": errs, "N_pos": ref.N_pos, "N_neg": ref.N_neg,
               "config": {"C": cfg.C, "d": d, "global_batch": N_loc * Wl, "M_glob": M * Wl,
                          "prefill_blocks": nblk, "s": cfg.s, "m": cfg.m},
               "bars": {"loss_rel": LOSS_RTOL, "dx_frac": DX_FRAC}}
    if world > 1:
        t = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.broadcast(t, 0)
        ok = int(t.item())
    return res if rank == 0 else {"ok": bool(ok)}


# --------------------------------------------------------------------------- roofline
def roofline_block(cfg, world, d, npos_avg, t_launch, ms_step, clocks, pk, share):
    """Roofline of the dominant kernel (dcp_pc_kernel) and of the whole step.
    Peak: burst when the median SM clock under load is within 5 % of its maximum, else the
    sustained (power-capped) figure; both fractions are reported."""
    C_loc = cfg.C // world
    burst = pk["bf16_tflops"]
    sus = pk.get("bf16_tflops_sustained", burst)
    near_max = (clocks is None or clocks.get("sm_max_mhz", 0) <= 0 or
                clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    peak = burst if near_max else sus
    flops_alg = 4.0 * npos_avg * C_loc * d          # GEMM 1 + GEMM 2 on the in-pool rows
    achieved = flops_alg / t_launch / 1e12
    # MMA rows: 128-row groups (TMEM lanes); a last group of <= 64 rows runs with M = 64
    # (dcp_pc_kernel's tail unit; evaluated at the average N_pos)
    full = math.floor(npos_avg / 128) * 128
    tail = npos_avg - full
    rows_exec = full + (0 if tail == 0 else 64 if tail <= 64 else 128)
    flops_exec = 4.0 * rows_exec * C_loc * d
    N = cfg.N_loc() * world
    # algorithmic bytes of one step per GPU: the pool read once, x in / dx out, the enqueue
    # (block read + slot write), the EMA (p, g read, g write); NVLink: C1 + C3 + C4 + C5
    hbm_bytes = C_loc * d * 2 + N * d * 2 * 2 + cfg.M_glob(world) * d * 2 * 2 + EMA_PARAMS * 12
    nvl_bytes = 0.0 if world == 1 else (N * d * 2 + N * 16 * world + N * d * 4 + cfg.M_glob(world) * d * 2) * (world - 1) / world
    t_roof = max(flops_alg / (burst * 1e12), hbm_bytes / (pk["hbm_gbs"] * 1e9), nvl_bytes / 900e9)
    traffic, traffic_src = None, None
    prof_file = os.path.join(ROOT, "profiles", f"ncu_main_{cfg.name}.json")
    if os.path.exists(prof_file):
        try:
            prof = json.load(open(prof_file))
            traffic = prof.get("dram_bytes_per_launch")
            traffic_src = f"profiles/ncu_main_{cfg.name}.json: {prof.get('source')}"
        except Exception:
            traffic, traffic_src = None, None
    # the decomposition's data movement into the SMs: every 128-row group streams the shard through
    # BOTH CTAs of its pair (producer: GEMM 1, consumer: GEMM 2) and ships P (32 KB per tile) over DSMEM.
    # Against the L2 -> SM TMA rate this chip sustains (profiles/r02_tma_l2_bench.txt): not the bound
    #
    groups = math.ceil(npos_avg / 128) if npos_avg > 0 else 0
    n_tiles = math.ceil(C_loc / 128)
    l2_bytes = groups * (2 * C_loc * d * 2 + n_tiles * 128 * 128 * 2)
    l2_peak = 20.9                         # TB/s, measured: 148 SMs TMA-streaming L2-resident 128-row boxes
    l2_ach = l2_bytes / t_launch / 1e12
    secondary = {"bound": "l2_to_sm", "achieved": l2_ach, "peak": l2_peak, "unit": "TB/s", "frac": l2_ach / l2_peak,
                 "bytes_per_launch": l2_bytes,
                 "peak_source": "scripts/tma_bench.cu on this B200: 148 CTAs streaming L2-resident [128 x 64] bf16 "
                                "SW128 TMA boxes, 20.1-20.9 TB/s (profiles/r02_tma_l2_bench.txt)",
                 "bytes_definition": "row groups x (2 CTAs x C_loc x d x 2 B pool tiles + tiles x 32 KB P over DSMEM)"}
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "dcp_pc_kernel (producer: TMEM-A logits GEMM + softmax -> DSMEM P; consumer: P x pool GEMM, O in TMEM)",
            "peak_kind": ("burst bf16 (median SM clock within 5 % of max)" if near_max else
                          "sustained bf16 (SM clock > 5 % below max: power-capped run)"),
            "peak_source": pk.get("_source"),
            "frac_vs_burst": achieved / burst, "frac_vs_sustained": achieved / sus,
            "algorithmic_flops_per_launch": flops_alg, "executed_mma_flops_per_launch": flops_exec,
            "tensor_pipe_frac": flops_exec / t_launch / 1e12 / peak,
            "avg_launch_ms": t_launch * 1e3, "N_pos_avg": npos_avg, "main_kernel_share_of_step": share,
            "step": {"t_roof_ms": t_roof * 1e3, "t_step_ms": ms_step, "frac": t_roof * 1e3 / ms_step,
                     "hbm_bytes": hbm_bytes, "nvlink_bytes": nvl_bytes,
                     "definition": "T_roof = max(F_alg / burst bf16, HBM bytes / measured copy BW, "
                                   "NVLink bytes / 900 GB/s); frac = T_roof / T_step (SURVEY 8(d))"},
            "secondary": secondary}


# --------------------------------------------------------------------------- GPU arm
def run_ours(args, cfg, world, rank, local_rank, device_only=False, cpu=True):
    import torch
    import torch.distributed as dist
    import paper_2105_10375_b200 as dcp

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    M, N_loc, d = cfg.M_loc, cfg.N_loc(), cfg.d
    uid = _nccl_uid(world, rank, dev)
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

    # ---- device-resident timed run (value): `trials` timed regions of exactly K steps each
    Ks, T = args.steps, max(1, args.trials)
    barrier()
    clk = Clocks(local_rank) if rank == 0 else None
    head.profile(True)
    launches[0] = 0
    trial_ms = []
    for _ in range(T):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.cuda.nvtx.range_push("timed_steps")  # ncu --nvtx-include timed_steps/ selects these launches
        for i in range(Ks):
            step(devin[i % R])
        join()
        torch.cuda.nvtx.range_pop()
        e1.record(stream)
        barrier()
        trial_ms.append(maxrank(e0.elapsed_time(e1)))
    clocks = clk.stop() if clk else None
    n_launch = launches[0] // T
    main_ms, main_n, npos_sum = head.profile_read()
    head.profile(False)
    if not timing_experiment:
        head.check()
    ms = statistics.median(trial_ms)
    value = Ks * N_loc * world / (ms / 1e3)
    best = Ks * N_loc * world / (min(trial_ms) / 1e3)
    npos_avg = npos_sum / max(1, main_n)
    t_launch = main_ms / max(1, main_n) / 1e3
    share = (main_ms / T) / ms
    pk = _peaks()
    roof = roofline_block(cfg, world, d, npos_avg, t_launch, ms / Ks, clocks, pk, share)
    trials = {"n": T, "ms_per_step": [t / Ks for t in trial_ms], "median_value": value, "best_value": best}

    if device_only:
        head.close()
        if rank != 0:
            return None
        return {"workload": cfg.name, "value": value, "unit": UNIT, "ms_per_step": ms / Ks, "trials": trials,
                "roofline": roof, "clocks": clocks, "config": _config(cfg, world, args.ema_overlap, args.K, _variant(args))}

    # ---- end-to-end through the public API with host buffers (e2e): every step copies its
    # inputs from pinned host memory and reads the loss back.  The copies run on a copy
    # stream into double-buffered device inputs, so step i+1's upload overlaps step i.
    loss_host = torch.zeros((), dtype=torch.float32).pin_memory()
    bufs = [tuple(torch.empty_like(a) for a in devin[0]) for _ in range(2)]
    copy_st = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    e2e_ms = []
    for _ in range(T):
        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        copy_st.wait_event(e2)                       # no upload before the timed region starts
        for i in range(Ks):
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
        e2e_ms.append(maxrank(e2.elapsed_time(e3)))
    if not timing_experiment:
        head.check()
    ms_e2e = statistics.median(e2e_ms)
    value_e2e = Ks * N_loc * world / (ms_e2e / 1e3)
    head.close()
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": Ks,
        "warmup": args.warmup, "ms_per_step": ms / Ks, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": _config(cfg, world, args.ema_overlap, args.K, _variant(args)),
        "trials": trials,
        "roofline": roof,
        "e2e": {"value": value_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": 4, "ms_per_step": ms_e2e / Ks,
                "trials_ms_per_step": [t / Ks for t in e2e_ms],
                "readback": "the fp32 loss scalar each step; dx (the backbone's input gradient) stays "
                            "on the device where the training step consumes it"},
        "gpu_launches": n_launch,
        "clocks": clocks,
    }
    if world == 1 and cpu and not args.no_cpu_baseline:
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
    # the block read, the overwritten rows read (their mu contributions leave, R3), the slot rows
    # and labels written; the label index's few random 8-B accesses per row are not counted
    byt = M * d * 2 * 3 + M * 8 * 2
    out["enqueue"] = {"rows": M, "bytes": byt, "best_ms": min(ts), "GBps": byt / (min(ts) * 1e-3) / 1e9,
                      "frac_of_measured_copy": byt / (min(ts) * 1e-3) / 1e9 / pk["hbm_gbs"]}
    head.close()
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


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n, argv):
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (one process per GPU)
    with the driver's own launcher form; rank 0 prints the line, and the exit code is the
    launcher's."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def dry_run(world, rank, local_rank):
    """--dry-run: the launch path only (process group, rank / world agreement); no kernels."""
    import torch
    import torch.distributed as dist
    if world > 1:
        use_nccl = torch.cuda.is_available() and torch.cuda.device_count() >= world
        if use_nccl:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, (rank, local_rank, os.getpid()))
        backend = dist.get_backend()
        dist.destroy_process_group()
    else:
        got, backend = [(0, 0, os.getpid())], None
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "backend": backend,
                          "ranks": [g[0] for g in got], "local_ranks": [g[1] for g in got],
                          "distinct_processes": len({g[2] for g in got})}), flush=True)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--trials", type=int, default=3, help="timed regions of --steps steps each (median, best)")
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
    ap.add_argument("--no-w-parity", action="store_true", help="skip the pre-timing self-check (debug only)")
    ap.add_argument("--dry-run", action="store_true", help="launch path only: ranks, world, backend")
    ap.add_argument("--kernel-bench", action="store_true", help="HBM-bound kernels alone (enqueue, EMA)")
    ap.add_argument("--sweep-c4", action="store_true", help="BJ:11 sweep, one rank of W=8 per point (evidence)")
    ap.add_argument("--also", default="c2", help="extra single-GPU workloads measured in the same run "
                    "(the north-star 1M-slot config c2 by default); 'none' to skip")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    in_launcher = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        # the CPU arm: rank 0 alone works (under torchrun the other ranks exit without work);
        # its config is the GPU arm's at N = --gpus ranks
        world = int(os.environ.get("WORLD_SIZE", args.gpus))
        if in_launcher and world != args.gpus:
            sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        if int(os.environ.get("RANK", "0")) == 0:
            run_reference(args, _workload(args.workload), world)
        return 0
    if args.gpus > 1 and not in_launcher:
        return spawn_ranks(args.gpus, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: {world} ranks launched but --gpus {args.gpus}: refusing to report a "
                 f"{world}-rank number as {args.gpus} GPUs")
    if args.dry_run:
        dry_run(world, rank, local_rank)
        return 0
    cfg = _workload(args.workload)
    if args.kernel_bench:
        kernel_bench(args)
        return 0
    if args.sweep_c4:
        sweep_c4(args)
        return 0
    import torch
    if world > 1:
        import torch.distributed as dist
        if torch.cuda.device_count() < world:
            sys.exit(f"bench.py: --gpus {world} but only {torch.cuda.device_count()} visible GPU(s)")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    wp = None
    if not args.no_w_parity:
        wp = w_parity(world, rank, local_rank, dev, emulate=0 if world > 1 else 2)
        if not wp["ok"]:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                                  "error": "w_parity self-check failed: no value reported", "w_parity": wp}),
                      flush=True)
            if world > 1:
                torch.distributed.destroy_process_group()
            return 1
    line = run_ours(args, cfg, world, rank, local_rank)
    extras = [w.strip("'\"") for w in args.also.split(",")]
    extras = [w for w in extras if w and w != "none" and w != args.workload] if world == 1 else []
    if extras:
        torch.cuda.empty_cache()
        line["also"] = []
        for w in extras:
            r = run_ours(args, _workload(w), world, rank, local_rank)
            torch.cuda.empty_cache()
            r = {k: v for k, v in r.items() if k not in ("metric", "higher_is_better", "scaling", "vs_baseline",
                                                        "data", "dtype", "n_gpus", "steps", "warmup")}
            line["also"].append({"workload": w, **r})
    if rank == 0 and line is not None:
        if wp is not None:
            line["w_parity"] = wp
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
