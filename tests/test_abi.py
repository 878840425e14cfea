"""The C-ABI library loads, exports every symbol include/packinfer.h declares, and validates its
arguments (no device compute here — CPU only)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pk = pytest.importorskip("paper_2602_06072_b200.packinfer")


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "packinfer.h")).read()
    return sorted(set(re.findall(r"PI_API\s+[\w\s\*]+?\b(packinfer_\w+)\s*\(", hdr)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) == 17, syms
    L = pk.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(pk.EXPORTS) <= set(syms)


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", pk._LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout


def test_strerror_and_version():
    L = pk.lib()
    assert L.packinfer_strerror(0) == b"ok"
    assert L.packinfer_strerror(-1) == b"invalid argument"
    assert b"sm_100a" in L.packinfer_version()


def test_plan_validation():
    with pytest.raises(pk.PackInferError) as e:
        pk.packinfer_plan([0], [1])
    assert e.value.status == pk.PI_EINVAL
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([5], [6])
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([10], [5], [0], [6])            # prefix would hold query rows
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([10], [5], [3], [2])            # prefix id out of range
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([10], [5], cfg=pk.default_config(tile_q=64))
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([10], [5], cfg=pk.default_config(decode_chunk=100))
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan([10], [5], cfg=pk.default_config(capacity=100, mem_cap=50))


def test_two_call_sizing_and_empty_batch():
    L = pk.lib()
    cfg = pk.default_config()
    out = pk.pi_plan()
    kv = np.array([10, 20], np.int32)
    st = L.packinfer_plan(2, kv.ctypes.data, kv.ctypes.data, None, 0, None, ctypes.byref(cfg), None, 0,
                          ctypes.byref(out))
    assert st == pk.PI_ENOSPC and out.arena_bytes > 0 and out.n_pieces == 2
    hp = pk.packinfer_plan([], [])
    assert hp.c.n_pieces == 0 and hp.c.n_groups == 0 and hp.c.buffer_tokens == 0
    assert hp.c.n_prefill_work == 0 and hp.c.n_decode_work == 0


def test_device_entry_points_validate_without_gpu():
    """NULL device plans are rejected before any device work."""
    L = pk.lib()
    assert L.packinfer_relayout_kv(None, None, None, None, 1, 128, 1, 0, 1, 64, 0, None, None, None) == pk.PI_EINVAL
    assert L.packinfer_attention_prefill(None, None, 0, None, None, 1, 1, 64, 0.0, 0, None, 0, None, None, None,
                                         None) == pk.PI_EINVAL
    assert L.packinfer_merge(None, None, None, 1, 64, 0, None, 0, None, None) == pk.PI_EINVAL
    # an empty plan makes every device call a no-op (no CUDA needed)
    dp = pk.pi_device_plan()
    assert L.packinfer_attention_decode(ctypes.byref(dp), None, 0, None, None, 1, 1, 64, 0.0, 0, None, 0, None,
                                        None, None, None) == pk.PI_OK
    assert L.packinfer_merge(ctypes.byref(dp), None, None, 1, 64, 0, None, 0, None, None) == pk.PI_OK
