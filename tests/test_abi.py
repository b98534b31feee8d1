"""CPU-side checks of the boundary: libf2c_dcp.so loads without a GPU and exports
every symbol include/f2c_dcp.h declares; host-side argument validation works
without launching anything."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "f2c_dcp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(f2c_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2105_10375_b200 import build
    build.build()
    import paper_2105_10375_b200 as m
    return m.load_library()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert {"f2c_dcp_create", "f2c_dcp_enqueue", "f2c_dcp_loss_fwd_bwd", "f2c_gnet_ema"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n


def test_state_bytes_and_validation_on_host(lib):
    sb = lib.f2c_dcp_state_bytes
    assert sb(1000, 512, 0, 1, 0, 1024, 512) > 1000 * 512 * 2
    assert sb(1000, 100, 0, 1, 0, 1024, 512) == 0          # d not a multiple of 128
    assert sb(1000, 512, 0, 2, 2, 1024, 512) == 0          # rank out of range
    one = sb(4096, 128, 0, 1, 0, 64, 64)
    two = sb(4096, 128, 0, 2, 0, 64, 64)
    assert two > 0 and sb(4096, 128, 0, 2, -1, 64, 64) >= 2 * (two - 1)  # emulated = W shards
    h = ctypes.c_void_p()
    # capacity check happens on the host before touching the device
    rc = lib.f2c_dcp_create(100, 128, 0, 1, 0, None, ctypes.c_void_p(256), 1 << 30, 16, 200,
                            ctypes.byref(h))
    assert rc == 3
    rc = lib.f2c_gnet_ema(None, None, 10, 1.5, None)
    assert rc == 1
    assert b"momentum" in lib.f2c_last_error()
