"""CPU fp64 oracle for the F2C DCP head -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2105_10375_b200``) never imports it and shares no code with it.

The arithmetic lives in ``f2c_oracle.c`` (plain C, fp64, single-threaded); this
module only compiles it with gcc and marshals numpy arrays through ctypes.
See the C file's header for the paper citations of each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "f2c_oracle.c")
_LIB = os.path.join(_HERE, "libf2c_oracle.so")

BF16, F32 = 0, 1
PHI_MEAN, PHI_SUM, PHI_MAX = 0, 1, 2   # NEXT-3 reductions of phi over the pool

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-std=c11", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.orc_enqueue.argtypes = [i64, i32, i32, P, P, P, P, P, P, i64]
        L.orc_enqueue_refresh.argtypes = [i64, i32, i32, P, P, P, P, P, P, i64, P]
        L.orc_loss.argtypes = [i64, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                               P, P, P, P, P, P, P, P, P]
        L.orc_loss_rows.argtypes = [i64, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                                    i64, P, P, P, P, P, P, P, P]
        L.orc_ema.argtypes = [P, P, i64, f64]
        L.orc_loss_k.argtypes = [i64, i32, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                                 P, P, P, P, P, P, P, P, P]
        L.orc_loss_rows_k.argtypes = [i64, i32, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                                      i64, P, P, P, P, P, P, P, P]
        L.orc_loss_v.argtypes = [i64, i32, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                                 i32, i32, f64, P, P, P, P, P, P, P, P, P]
        L.orc_loss_rows_v.argtypes = [i64, i32, i32, i32, P, P, i64, i64, i64, P, P, P, f64, f64,
                                      i32, i32, f64, i64, P, P, P, P, P, P, P, P]
        for f in (L.orc_enqueue, L.orc_enqueue_refresh, L.orc_loss, L.orc_loss_rows, L.orc_ema, L.orc_loss_k,
                  L.orc_loss_rows_k, L.orc_loss_v, L.orc_loss_rows_v):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _raw_dtype(arr: np.ndarray) -> int:
    if arr.dtype == np.uint16:
        return BF16
    if arr.dtype == np.float32:
        return F32
    raise TypeError(f"oracle inputs must be bf16 bit patterns (uint16) or float32, got {arr.dtype}")


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle error code {code}")
        self.code = code


@dataclass
class LossResult:
    L: float
    L_ce: float
    L_cos: float
    dx: np.ndarray      # [N, d] float64
    lse: np.ndarray     # [N]
    tslot: np.ndarray   # [N] int64, -1 = out of pool
    phi: np.ndarray     # [N]
    ell: np.ndarray     # [N]
    N_pos: int
    N_neg: int
    C_occ: int
    P: np.ndarray | None = None
    dT: np.ndarray | None = None


class Pool:
    """The DCP state of the oracle: T [C, d] (K = 1) or [C, K, d] (raw dtype), lab [C], E,
    M_last.  An enqueued identity carries K features."""

    def __init__(self, C: int, d: int, dtype: int = BF16, K: int = 1):
        self.C, self.d, self.dtype, self.K = int(C), int(d), int(dtype), int(K)
        shape = (C, d) if K == 1 else (C, K, d)
        self.T = np.zeros(shape, dtype=np.uint16 if dtype == BF16 else np.float32)
        self.lab = np.full(C, -1, dtype=np.int64)
        self.E = np.zeros(1, dtype=np.int64)
        self.M_last = np.zeros(1, dtype=np.int64)
        # after a refresh-in-place enqueue (NEXT-3): write index of the slot holding each row
        # of the last block (the pairing check's target); None after a pure Eq. 7 enqueue
        self.blk_seq = None

    @property
    def C_occ(self) -> int:
        return int(min(self.E[0], self.C))

    def enqueue(self, G: np.ndarray, y: np.ndarray, refresh: bool = False) -> None:
        """Eq. 7 / Algorithm 1 (orc_enqueue); refresh=True: SPEC's refresh-in-place insert
        (orc_enqueue_refresh, NEXT-3, reading R7)."""
        G = np.ascontiguousarray(G)
        y = np.ascontiguousarray(y, dtype=np.int64)
        want = (len(y), self.d) if self.K == 1 else (len(y), self.K, self.d)
        if _raw_dtype(G) != self.dtype or G.shape != want:
            raise OracleError(2, "enqueue shape/dtype")
        # a slot holds K consecutive feature rows: the ring copy is the same with rows of K*d
        if refresh:
            bs = np.zeros(len(y), dtype=np.int64)
            rc = lib().orc_enqueue_refresh(self.C, self.K * self.d, self.dtype, _p(self.T), _p(self.lab),
                                           _p(self.E), _p(self.M_last), _p(G), _p(y), len(y), _p(bs))
            if rc:
                raise OracleError(rc, "orc_enqueue_refresh")
            self.blk_seq = bs
            return
        rc = lib().orc_enqueue(self.C, self.K * self.d, self.dtype, _p(self.T), _p(self.lab), _p(self.E),
                               _p(self.M_last), _p(G), _p(y), len(y))
        if rc:
            raise OracleError(rc, "orc_enqueue")
        self.blk_seq = None

    def _pairing(self, pairing, tslot):
        """The C oracle checks pairing against the pure ring (E - M_last + j); after a
        refresh enqueue row j's slot is blk_seq[j] mod C instead (D13 with R7)."""
        if pairing is None or self.blk_seq is None:
            return pairing
        pr = np.asarray(pairing)
        for i in np.where(pr >= 0)[0]:
            j = int(pr[i])
            if j >= int(self.M_last[0]) or tslot[i] != self.blk_seq[j] % self.C:
                raise OracleError(4, "orc_loss pairing")
        return None

    def loss(self, X: np.ndarray, y: np.ndarray, pairing: np.ndarray | None, s: float, m: float,
             want_P: bool = False, want_dT: bool = False, phi_mode: int = PHI_MEAN,
             hinge: bool = False, lam: float = 1.0, excl_dup: bool = False) -> LossResult:
        X = np.ascontiguousarray(X)
        y = np.ascontiguousarray(y, dtype=np.int64)
        N, d = len(y), self.d
        if _raw_dtype(X) != self.dtype or X.shape != (N, d):
            raise OracleError(2, "loss shape/dtype")
        pr = None if pairing is None else np.ascontiguousarray(pairing, dtype=np.int32)
        pr_after = pr if self.blk_seq is not None else None
        if pr_after is not None:
            pr = None
        out3 = np.zeros(3)
        dx = np.zeros((N, d))
        lse, phi, ell = np.zeros(N), np.zeros(N), np.zeros(N)
        ts = np.zeros(N, dtype=np.int64)
        counts = np.zeros(3, dtype=np.int64)
        P = np.zeros((N, self.C_occ)) if want_P else None
        dT = np.zeros((self.C, d)) if want_dT else None
        rc = lib().orc_loss_v(self.C, self.K, d, self.dtype, _p(self.T), _p(self.lab),
                              int(self.E[0]), int(self.M_last[0]), N, _p(X), _p(y), _p(pr),
                              float(s), float(m), int(phi_mode), int(bool(hinge)) | (int(bool(excl_dup)) << 1),
                              float(lam), _p(out3), _p(dx), _p(lse), _p(ts), _p(phi), _p(ell), _p(counts),
                              _p(P), _p(dT))
        if rc:
            raise OracleError(rc, "orc_loss")
        self._pairing(pr_after, ts)
        return LossResult(out3[0], out3[1], out3[2], dx, lse, ts, phi, ell,
                          int(counts[0]), int(counts[1]), int(counts[2]), P, dT)

    def loss_rows(self, X, y, pairing, s, m, rows, phi_mode: int = PHI_MEAN, hinge: bool = False,
                  lam: float = 1.0, excl_dup: bool = False):
        X = np.ascontiguousarray(X)
        y = np.ascontiguousarray(y, dtype=np.int64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        N, d, k = len(y), self.d, len(rows)
        pr = None if pairing is None else np.ascontiguousarray(pairing, dtype=np.int32)
        if self.blk_seq is not None and pr is not None:
            self.loss(X, y, pr, s, m, phi_mode=phi_mode, hinge=hinge, lam=lam, excl_dup=excl_dup)
            pr = None   # (checked above over the whole batch)
        dx = np.zeros((k, d))
        lse, phi, ell = np.zeros(k), np.zeros(k), np.zeros(k)
        ts = np.zeros(k, dtype=np.int64)
        counts = np.zeros(3, dtype=np.int64)
        mu = np.zeros(d)
        rc = lib().orc_loss_rows_v(self.C, self.K, d, self.dtype, _p(self.T), _p(self.lab),
                                   int(self.E[0]), int(self.M_last[0]), N, _p(X), _p(y), _p(pr),
                                   float(s), float(m), int(phi_mode),
                                   int(bool(hinge)) | (int(bool(excl_dup)) << 1), float(lam),
                                   k, _p(rows), _p(dx), _p(lse), _p(ts),
                                   _p(phi), _p(ell), _p(counts), _p(mu))
        if rc:
            raise OracleError(rc, "orc_loss_rows")
        return dict(dx=dx, lse=lse, tslot=ts, phi=phi, ell=ell, N_pos=int(counts[0]),
                    N_neg=int(counts[1]), C_occ=int(counts[2]), mu=mu)


def ema(p: np.ndarray, g: np.ndarray, momentum: float) -> np.ndarray:
    """Returns the updated copy of g (fp32), g <- m g + (1-m) p in fp64."""
    p = np.ascontiguousarray(p, dtype=np.float32)
    out = np.array(g, dtype=np.float32, copy=True)
    rc = lib().orc_ema(_p(p), _p(out), out.size, float(momentum))
    if rc:
        raise OracleError(rc, "orc_ema")
    return out


def bf16_to_f64(a: np.ndarray) -> np.ndarray:
    """Exact upcast of bf16 bit patterns (uint16) to float64."""
    return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f64_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float64 values to bf16 (nearest-even), returned as uint16 bit patterns.

    Only used by tests to build small hand-made fixtures; the synthetic workload
    generator has its own rounding in synth/.
    """
    a = np.asarray(a, dtype=np.float64)
    m, e = np.frexp(a)                     # a = m * 2**e, |m| in [0.5, 1)
    q = np.rint(m * 256.0)                 # 8 significant bits, ties to even
    v = np.ldexp(q, e - 8).astype(np.float32)  # exact in fp32
    return (v.view(np.uint32) >> 16).astype(np.uint16)
