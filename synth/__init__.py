"""Seeded synthetic workloads shaped like the paper's.

This module serves both the oracle tests and the CUDA path.  It holds none of
the method's arithmetic: ``f2c_synth.c`` draws counter-based random numbers,
normalises generated vectors and rounds them to the input dtype.

Configurations c0-c4 follow BASELINE.json ``configs`` (BJ:7-11).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "f2c_synth.c")
_LIB = os.path.join(_HERE, "libf2c_synth.so")

BF16, F32 = 0, 1
SEED_BASE = 210510375

# RNG stream ids
S_PRE, S_PRE_LAB, S_INST, S_INST_LAB, S_IDX, S_IDN, S_EMA_P, S_EMA_G = 1, 2, 3, 4, 5, 6, 8, 9

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=c11", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, i64, i32, f64, P = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                 ctypes.c_void_p)
        L.syn_gauss.argtypes = [u64, u64, u64, i64, i64, i32, P]
        L.syn_unit_rows.argtypes = [u64, u64, u64, i64, i64, i32, i32, P]
        L.syn_pair_rows.argtypes = [u64, u64, u64, u64, i64, i64, i32, f64, i32, P, P]
        L.syn_uniform_labels.argtypes = [u64, u64, u64, i64, i64, i64, P]
        L.syn_identity_labels.argtypes = [u64, u64, i64, i64, i64, i64, P]
        L.syn_f32_normal.argtypes = [u64, u64, i64, i64, f64, P]
        for f in (L.syn_gauss, L.syn_unit_rows, L.syn_pair_rows, L.syn_uniform_labels,
                  L.syn_identity_labels, L.syn_f32_normal):
            f.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _np_dtype(dtype):
    return np.uint16 if dtype == BF16 else np.float32


def gauss(seed, stream, step, row0, nrows, d):
    out = np.empty((nrows, d), dtype=np.float64)
    lib().syn_gauss(seed, stream, step, row0, nrows, d, _p(out))
    return out


def unit_rows(seed, stream, step, row0, nrows, d, dtype=BF16):
    out = np.empty((nrows, d), dtype=_np_dtype(dtype))
    if nrows:
        lib().syn_unit_rows(seed, stream, step, row0, nrows, d, dtype, _p(out))
    return out


def pair_rows(seed, step, row0, nrows, d, sigma, dtype=BF16):
    x = np.empty((nrows, d), dtype=_np_dtype(dtype))
    g = np.empty((nrows, d), dtype=_np_dtype(dtype))
    if nrows:
        lib().syn_pair_rows(seed, S_IDX, S_IDN, step, row0, nrows, d, float(sigma), dtype, _p(x),
                            _p(g))
    return x, g


def uniform_labels(seed, stream, step, row0, n, n_id):
    out = np.empty(n, dtype=np.int64)
    if n:
        lib().syn_uniform_labels(seed, stream, step, row0, n, n_id, _p(out))
    return out


def identity_labels(seed, block, row0, n, M_glob, n_id):
    out = np.empty(n, dtype=np.int64)
    if n:
        lib().syn_identity_labels(seed, block, row0, n, M_glob, n_id, _p(out))
    return out


def f32_normal(seed, stream, n, sigma, off=0):
    assert off % 1024 == 0
    out = np.empty(n, dtype=np.float32)
    lib().syn_f32_normal(seed, stream, off, n, float(sigma), _p(out))
    return out


@dataclass(frozen=True)
class Config:
    """One workload of BASELINE.json (BJ:7-11). M_loc = identity rows per rank per step;
    the per-rank P-Net batch is N_loc = 2*M_loc (M_loc instance + M_loc identity rows)."""
    name: str
    d: int
    C: int
    M_loc: int
    n_id: int
    dtype: int
    s: float = 64.0
    m: float = 0.35
    sigma: float = 0.3           # per-coordinate pair noise (D18, literal reading)
    prefill: int = 0             # number of prefill enqueues (D20); 0 = ceil(C / M_glob)
    steps: int = 20
    seed: int = SEED_BASE

    def N_loc(self):
        return 2 * self.M_loc

    def M_glob(self, world=1):
        return self.M_loc * world

    def prefill_blocks(self, world=1):
        return max(self.prefill, math.ceil(self.C / self.M_glob(world)))


CONFIGS = {
    # BJ:7 tiny CPU-seconds case (fp32 inputs; D21)
    "c0": Config("c0", d=128, C=1024, M_loc=64, n_id=10_000, dtype=F32, prefill=16, steps=20,
                 seed=SEED_BASE + 0),
    # BJ:8 single-GPU mid size, pool warmed by 200 enqueues
    "c1": Config("c1", d=512, C=100_000, M_loc=512, n_id=10_000_000, dtype=BF16, prefill=200,
                 steps=100, seed=SEED_BASE + 1),
    # BJ:9 single-GPU large pool (1M slots, 10 % of 10M ids)
    "c2": Config("c2", d=512, C=1_048_576, M_loc=1024, n_id=10_000_000, dtype=BF16, steps=100,
                 seed=SEED_BASE + 2),
    # BJ:10 sharded 4M-slot pool, per-GPU M=512 (global batch 1024*W)
    "c3": Config("c3", d=512, C=4_194_304, M_loc=512, n_id=80_000_000, dtype=BF16, steps=100,
                 seed=SEED_BASE + 3),
}


def c4_point(C_frac: float, N_glob: int, world: int = 8) -> Config:
    """BJ:11 sweep point: C = C_frac * 10M, global batch N_glob over `world` ranks."""
    return Config(f"c4_C{int(C_frac * 100)}_N{N_glob}", d=512, C=int(C_frac * 10_000_000),
                  M_loc=N_glob // (2 * world), n_id=10_000_000, dtype=BF16, steps=100,
                  seed=SEED_BASE + 4)


def scaled(cfg: Config, **kw) -> Config:
    return replace(cfg, **kw)


def prefill_block(cfg: Config, b: int, rank: int = 0, world: int = 1):
    """Prefill enqueue b (D20): normalised Gaussian rows with i.i.d. uniform labels.
    Returns this rank's part (rows [rank*M_loc, (rank+1)*M_loc) of the global block)."""
    r0 = rank * cfg.M_loc
    g = unit_rows(cfg.seed, S_PRE, b, r0, cfg.M_loc, cfg.d, cfg.dtype)
    y = uniform_labels(cfg.seed, S_PRE_LAB, b, r0, cfg.M_loc, cfg.n_id)
    return g, y


@dataclass
class Step:
    x: np.ndarray        # [N_loc, d] P-Net rows (instance rows first, then identity rows)
    y: np.ndarray        # [N_loc] labels
    pairing: np.ndarray  # [N_loc] int32: -1 instance row, else row of the global enqueue block
    g: np.ndarray        # [M_loc, d] G-Net features of this rank's identity rows (enqueued)
    gy: np.ndarray       # [M_loc] identity labels (distinct within the global block)


def step_inputs(cfg: Config, t: int, rank: int = 0, world: int = 1, sigma: float | None = None) -> Step:
    """Mixed batch of step t for `rank`: M_loc instance rows with uniform
    labels (I) and M_loc identity rows (III) whose G-Net pairs (IV) are enqueued."""
    sigma = cfg.sigma if sigma is None else sigma
    M, d, Mg = cfg.M_loc, cfg.d, cfg.M_glob(world)
    r0 = rank * M
    xi = unit_rows(cfg.seed, S_INST, t, r0, M, d, cfg.dtype)
    yi = uniform_labels(cfg.seed, S_INST_LAB, t, r0, M, cfg.n_id)
    xd, g = pair_rows(cfg.seed, t, r0, M, d, sigma, cfg.dtype)
    yd = identity_labels(cfg.seed, t, r0, M, Mg, cfg.n_id)
    x = np.concatenate([xi, xd], axis=0)
    y = np.concatenate([yi, yd])
    pairing = np.concatenate([np.full(M, -1, np.int32), (r0 + np.arange(M)).astype(np.int32)])
    return Step(x=x, y=y, pairing=pairing, g=g, gy=yd)


def sigma_regime(name: str, d: int) -> float:
    """Pair-noise regimes of D18: literal per-coordinate 0.3, balanced (total 1.25),
    peaked (total 0.3)."""
    return {"literal": 0.3, "balanced": 1.25 / math.sqrt(d), "peaked": 0.3 / math.sqrt(d)}[name]
