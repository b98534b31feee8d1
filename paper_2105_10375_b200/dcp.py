"""ctypes binding of libf2c_dcp.so (same names as include/f2c_dcp.h) and a small
torch-facing wrapper.  Argument marshalling only; no arithmetic of the method."""
from __future__ import annotations

import ctypes
import os

import torch

BF16, F32 = 0, 1
PHI_MEAN, PHI_SUM, PHI_MAX = 0, 1, 2
_HERE = os.path.dirname(os.path.abspath(__file__))
# F2C_LIB overrides the library path (A/B timing experiments only; the default is in-tree)
lib_path = os.environ.get("F2C_LIB") or os.path.join(_HERE, "libf2c_dcp.so")

STATUS = {0: "F2C_OK", 1: "F2C_EINVAL", 2: "F2C_ESHAPE", 3: "F2C_ECAPACITY", 4: "F2C_EPAIRING",
          5: "F2C_ECUDA", 6: "F2C_ENCCL", 7: "F2C_EDEVICE"}

_lib = None


class DCPError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load_library():
    """Load the in-tree libf2c_dcp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} not built; run paper_2105_10375_b200/build.py (or "
                          "__graft_entry__.build())")
    L = ctypes.CDLL(lib_path)
    P, i64, i32, f32, f64, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float,
                                 ctypes.c_double, ctypes.c_size_t)
    L.f2c_dcp_state_bytes.argtypes = [i64, i32, i32, i32, i32, i64, i64]
    L.f2c_dcp_state_bytes.restype = sz
    L.f2c_dcp_create.argtypes = [i64, i32, i32, i32, i32, P, P, sz, i64, i64, ctypes.POINTER(P)]
    L.f2c_dcp_state_bytes_k.argtypes = [i64, i32, i32, i32, i32, i32, i64, i64]
    L.f2c_dcp_state_bytes_k.restype = sz
    L.f2c_dcp_create_k.argtypes = [i64, i32, i32, i32, i32, i32, P, P, sz, i64, i64, ctypes.POINTER(P)]
    L.f2c_dcp_enqueue.argtypes = [P, P, P, i64, P]
    L.f2c_dcp_loss_fwd_bwd.argtypes = [P, P, P, P, i64, f32, f32, P, P, P]
    L.f2c_gnet_ema.argtypes = [P, P, i64, f64, P]
    L.f2c_dcp_get_state.argtypes = [P, P, P, P]
    L.f2c_dcp_set_state.argtypes = [P, P, P, i64]
    L.f2c_dcp_row_stats.argtypes = [P, P, P, P, P, P, P]
    L.f2c_dcp_check.argtypes = [P]
    L.f2c_last_error.argtypes = []
    L.f2c_last_error.restype = ctypes.c_char_p
    L.f2c_last_launch_count.argtypes = []
    L.f2c_dcp_profile.argtypes = [P, i32]
    L.f2c_dcp_profile_read.argtypes = [P, P, P, P]
    L.f2c_dcp_fused_kernel.argtypes = [P, i64, P, P]
    L.f2c_dcp_destroy.argtypes = [P]
    L.f2c_dcp_destroy.restype = None
    L.f2c_dcp_set_lcos.argtypes = [P, i32, i32, ctypes.c_double]
    L.f2c_dcp_set_dup_mode.argtypes = [P, i32]
    L.f2c_dcp_set_enqueue_mode.argtypes = [P, i32]
    for f in (L.f2c_dcp_create, L.f2c_dcp_create_k, L.f2c_dcp_set_lcos, L.f2c_dcp_set_dup_mode,
              L.f2c_dcp_set_enqueue_mode, L.f2c_dcp_enqueue, L.f2c_dcp_loss_fwd_bwd, L.f2c_gnet_ema,
              L.f2c_dcp_get_state, L.f2c_dcp_set_state, L.f2c_dcp_row_stats, L.f2c_dcp_check,
              L.f2c_last_launch_count, L.f2c_dcp_profile, L.f2c_dcp_profile_read, L.f2c_dcp_fused_kernel):
        f.restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise DCPError(rc, load_library().f2c_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _tdtype(dtype):
    return torch.bfloat16 if dtype == BF16 else torch.float32


class DCPHead:
    """One rank's handle of the DCP (or an emulated world when rank == -1).

    The caller-owned state buffer is a torch uint8 CUDA tensor sized by
    f2c_dcp_state_bytes; all device memory comes from torch."""

    def __init__(self, C: int, d: int, dtype: int = BF16, world: int = 1, rank: int = 0,
                 n_local_max: int = 1024, m_local_max: int = 512, nccl_uid: bytes | None = None,
                 device=None, K: int = 1):
        L = load_library()
        if not torch.cuda.is_available():
            raise DCPError(5, "no CUDA device: the DCP head has no CPU path")
        self.C, self.d, self.dtype, self.world, self.rank = int(C), int(d), int(dtype), world, rank
        self.n_local_max, self.m_local_max, self.K = int(n_local_max), int(m_local_max), int(K)
        nbytes = L.f2c_dcp_state_bytes_k(C, K, d, dtype, world, rank, n_local_max, m_local_max)
        if nbytes == 0:
            raise DCPError(1, "invalid configuration for f2c_dcp_state_bytes")
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.state = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._h = ctypes.c_void_p()
        uid = None if nccl_uid is None else ctypes.create_string_buffer(bytes(nccl_uid), 128)
        _check(L.f2c_dcp_create_k(C, K, d, dtype, world, rank, uid, _ptr(self.state), nbytes,
                                  n_local_max, m_local_max, ctypes.byref(self._h)))

    # -- argument checks (marshalling only: shapes, dtypes, layout, device) ------------------
    def _rows_per_rank(self):
        return self.world if self.rank < 0 else 1

    def _check_tensor(self, t, name, dtype, shape=None):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor")
        if t.dtype != dtype:
            raise DCPError(1, f"{name}: dtype {t.dtype}, expected {dtype}")
        if t.device.type != "cuda" or (self.device.index is not None and t.device.index != self.device.index):
            raise DCPError(1, f"{name}: on {t.device}, the handle is on {self.device}")
        if not t.is_contiguous():
            raise DCPError(1, f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise DCPError(2, f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")

    # -- the hot path -----------------------------------------------------------------
    def enqueue(self, g_feats: torch.Tensor, labels: torch.Tensor, stream=None):
        """Eq. 7 / Algorithm 1: g_feats [m, d] (K = 1) or [m, K, d] in the handle's dtype, labels
        int64 [m] (an emulated world passes the rank-ordered global block, m = world * m_local)."""
        m = labels.shape[0] if labels.dim() == 1 else -1
        self._check_tensor(labels, "labels", torch.int64, (m,))
        want = (m, self.d) if self.K == 1 else (m, self.K, self.d)
        self._check_tensor(g_feats, "g_feats", _tdtype(self.dtype), want)
        if m % self._rows_per_rank():
            raise DCPError(2, f"emulated world: {m} block rows not divisible by world {self.world}")
        _check(load_library().f2c_dcp_enqueue(self._h, _ptr(g_feats), _ptr(labels), m // self._rows_per_rank(),
                                              _stream(stream)))

    def loss_fwd_bwd(self, x: torch.Tensor, labels: torch.Tensor, pairing: torch.Tensor | None,
                     s: float, m: float, dx: torch.Tensor | None = None, loss: torch.Tensor | None = None,
                     stream=None):
        """Returns (loss [fp32 device scalar], dx [same shape/dtype as x]).  Without `loss` a fresh
        device scalar is returned per call (it is written asynchronously on the stream)."""
        n = x.shape[0] if x.dim() == 2 else -1
        self._check_tensor(x, "x", _tdtype(self.dtype), (n, self.d))
        self._check_tensor(labels, "labels", torch.int64, (n,))
        if pairing is not None:
            self._check_tensor(pairing, "pairing", torch.int32, (n,))
        if n % self._rows_per_rank():
            raise DCPError(2, f"emulated world: {n} batch rows not divisible by world {self.world}")
        dx = torch.empty_like(x) if dx is None else dx
        self._check_tensor(dx, "dx", x.dtype, tuple(x.shape))
        loss = torch.empty((), dtype=torch.float32, device=x.device) if loss is None else loss
        self._check_tensor(loss, "loss", torch.float32)
        if loss.numel() != 1:
            raise DCPError(2, "loss must hold one fp32 element")
        n_local = n // self._rows_per_rank()
        _check(load_library().f2c_dcp_loss_fwd_bwd(self._h, _ptr(x), _ptr(labels), _ptr(pairing),
                                                   n_local, float(s), float(m), _ptr(loss), _ptr(dx),
                                                   _stream(stream)))
        return loss, dx

    def set_lcos(self, phi_mode: int = PHI_MEAN, hinge: bool = False, lam: float = 1.0):
        """NEXT-3 L_cos variant for later loss calls: phi_mode PHI_MEAN / PHI_SUM / PHI_MAX,
        hinge max(0, cos), L = L_ce + lam * L_cos (include/f2c_dcp.h)."""
        _check(load_library().f2c_dcp_set_lcos(self._h, int(phi_mode), int(hinge), float(lam)))

    def set_enqueue_mode(self, refresh_in_place: bool = False):
        """NEXT-3: SPEC's refresh-in-place enqueue (resident ids overwritten in place, age kept;
        reading R7) for later enqueues; False restores pure Eq. 7 (include/f2c_dcp.h)."""
        _check(load_library().f2c_dcp_set_enqueue_mode(self._h, int(bool(refresh_in_place))))

    def set_dup_mode(self, exclude_stale: bool = False):
        """NEXT-3: drop each in-pool row's stale self-duplicates (older slots of its own label)
        from its softmax in later loss calls; False restores reading D8 (include/f2c_dcp.h)."""
        _check(load_library().f2c_dcp_set_dup_mode(self._h, int(bool(exclude_stale))))

    # -- support ----------------------------------------------------------------------
    def check(self):
        _check(load_library().f2c_dcp_check(self._h))

    def get_state(self):
        import numpy as np
        rows = self.C if (self.rank < 0 or self.world == 1) else None
        if rows is None:
            lo = self.C * self.rank // self.world
            hi = self.C * (self.rank + 1) // self.world
            rows = hi - lo
        shape = (rows, self.d) if self.K == 1 else (rows, self.K, self.d)
        feats = np.empty(shape, dtype=np.uint16 if self.dtype == BF16 else np.float32)
        labs = np.empty(rows, dtype=np.int64)
        E = ctypes.c_int64()
        _check(load_library().f2c_dcp_get_state(self._h, feats.ctypes.data_as(ctypes.c_void_p),
                                                labs.ctypes.data_as(ctypes.c_void_p), ctypes.byref(E)))
        return feats, labs, E.value

    def _shard_rows(self):
        if self.rank < 0 or self.world == 1:
            return self.C
        return self.C * (self.rank + 1) // self.world - self.C * self.rank // self.world

    def set_state(self, feats, labels, E: int):
        """Restore this handle's slots (host arrays as get_state returns them: feats uint16 bf16
        bits or float32, [rows, d] or [rows, K, d]; labels int64 [rows], -1 = empty)."""
        import numpy as np
        feats = np.ascontiguousarray(feats)
        labels = np.ascontiguousarray(labels)
        rows = self._shard_rows()
        want = (rows, self.d) if self.K == 1 else (rows, self.K, self.d)
        want_dt = np.uint16 if self.dtype == BF16 else np.float32
        if feats.dtype != want_dt or feats.shape != want:
            raise DCPError(2, f"set_state feats: {feats.dtype}{feats.shape}, expected {np.dtype(want_dt)}{want}")
        if labels.dtype != np.int64 or labels.shape != (rows,):
            raise DCPError(2, f"set_state labels: {labels.dtype}{labels.shape}, expected int64({rows},)")
        _check(load_library().f2c_dcp_set_state(self._h, feats.ctypes.data_as(ctypes.c_void_p),
                                                labels.ctypes.data_as(ctypes.c_void_p), int(E)))

    # -- checkpoint / resume: this rank's shard of the pool, as a file --------
    def save(self, path: str):
        """Write this handle's pool state (features as stored, labels, E) and its geometry to an
        .npz file; one file per rank (a world > 1 job saves every rank's shard)."""
        import numpy as np
        feats, labs, E = self.get_state()
        np.savez(path, feats=feats, labels=labs, E=np.int64(E),
                 geometry=np.array([self.C, self.d, self.dtype, self.K, self.world, self.rank], dtype=np.int64))

    def load(self, path: str):
        """Restore a pool written by save() into a handle of the same geometry (C, d, dtype, K,
        world, rank); raises DCPError(F2C_ESHAPE) on a mismatch."""
        import numpy as np
        z = np.load(path)
        geo = [self.C, self.d, self.dtype, self.K, self.world, self.rank]
        if z["geometry"].tolist() != geo:
            raise DCPError(2, f"checkpoint geometry {z['geometry'].tolist()} != handle {geo}")
        self.set_state(z["feats"], z["labels"], int(z["E"]))

    def row_stats(self, n_global: int):
        import numpy as np
        lse, cos, phi, ell = (np.empty(n_global, np.float32) for _ in range(4))
        tseq = np.empty(n_global, np.int64)
        counts = np.empty(3, np.int64)
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _check(load_library().f2c_dcp_row_stats(self._h, P(lse), P(tseq), P(cos), P(phi), P(ell),
                                                P(counts)))
        return dict(lse=lse, target_seq=tseq, cos_t=cos, phi=phi, ell=ell, N_pos=int(counts[0]),
                    N_neg=int(counts[1]), C_occ=int(counts[2]))

    def profile(self, enable: bool):
        _check(load_library().f2c_dcp_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        ms, n, npos = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _check(load_library().f2c_dcp_profile_read(self._h, ctypes.byref(ms), ctypes.byref(n),
                                                   ctypes.byref(npos)))
        return ms.value, n.value, npos.value

    def fused_kernel(self, n_global: int):
        """(kind, ctas) of the fused loss kernel a call with n_global rows runs: kind 0 =
        dcp_pc_kernel, 1 = dcp_tp64_kernel, 2 = dcp_pc4_kernel (include/f2c_dcp.h)."""
        k, c = ctypes.c_int32(), ctypes.c_int32()
        _check(load_library().f2c_dcp_fused_kernel(self._h, n_global, ctypes.byref(k), ctypes.byref(c)))
        return k.value, c.value

    @staticmethod
    def last_launch_count() -> int:
        return load_library().f2c_last_launch_count()

    def close(self):
        if self._h:
            load_library().f2c_dcp_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id(device=None) -> bytes | None:
    """The 128-byte NCCL unique id a world > 1 DCPHead needs (f2c_dcp_create): made by rank 0 and
    broadcast over the default torch.distributed process group (plumbing only); None for world 1."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dist.get_rank() == 0:
        t = torch.tensor(list(bytes(torch.cuda.nccl.unique_id())), dtype=torch.uint8, device=dev)
    else:
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def gnet_ema(p: torch.Tensor, g: torch.Tensor, momentum: float, stream=None):
    """In-place g <- m g + (1-m) p (fp32, fp64 arithmetic, bit-exact)."""
    for name, t in (("p", p), ("g", g)):
        if t.dtype != torch.float32 or t.device.type != "cuda" or not t.is_contiguous():
            raise DCPError(1, f"gnet_ema {name}: contiguous fp32 CUDA tensor required")
    if p.numel() != g.numel() or p.device != g.device:
        raise DCPError(2, "gnet_ema: p and g must have the same size and device")
    _check(load_library().f2c_gnet_ema(_ptr(p), _ptr(g), g.numel(), float(momentum), _stream(stream)))
