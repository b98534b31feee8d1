"""Shared test helpers: build the same seeded workload for the GPU path and the
oracle, and compare results with the tolerances of BASELINE.json (BJ:5)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

LOSS_RTOL = 2e-3      # |L_gpu - L| <= 2e-3 |L|            (BJ:5)
DX_FRAC = 1e-2        # max|dx_gpu - dx| <= 1e-2 max|dx|     (BJ:5)


def to_dev(a: np.ndarray, dtype: int) -> torch.Tensor:
    if dtype == synth.BF16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def from_dev(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return oracle.bf16_to_f64(t.view(torch.int16).cpu().numpy().view(np.uint16))
    return t.double().cpu().numpy()


def lt(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def it(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def assert_loss_close(gpu: float, ref: float, rtol=LOSS_RTOL, atol=1e-6, what="loss"):
    assert abs(gpu - ref) <= rtol * abs(ref) + atol, f"{what}: gpu {gpu!r} oracle {ref!r}"


def assert_dx_close(dx_gpu: np.ndarray, dx_ref: np.ndarray, frac=DX_FRAC, what="dx"):
    scale = np.abs(dx_ref).max()
    err = np.abs(dx_gpu - dx_ref).max()
    assert err <= frac * scale + 1e-12, f"{what}: max err {err:.3e} > {frac} * max|dx| {scale:.3e}"


def assert_dx_rows_close(dx_gpu, dx_ref, rows, frac=DX_FRAC, what="dx"):
    """The BJ:5 criterion applied separately to a subset of rows (e.g. the in-pool or
    the out-of-pool rows, whose gradients differ by orders of magnitude)."""
    if len(rows) == 0:
        return
    assert_dx_close(dx_gpu[rows], dx_ref[rows], frac, what)
