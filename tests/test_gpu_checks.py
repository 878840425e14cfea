"""Debug build with device-side bounds checks (-DPI_CHECKS=1: every work item, span, row, partial
slot and head index the kernels dereference is checked; a failure prints its id and traps).
compute-sanitizer is closed on this GPU pool, so these checks stand in for it: the checked library
runs representative batches (prefill, decode loop, packed decode items, splits with partials, head
slices, in-kernel merge, d = 64, configs[3] at full size) without a trap and bitwise equal to the
production library."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_checked_build_no_trap_and_bitwise(tmp_path):
    from paper_2602_06072_b200 import build as B
    lib = os.path.join(ROOT, "variants", "libpi_checks.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    B.build(True, False, lib, ("PI_CHECKS=1",))
    outs = {}
    for name, path in (("checked", lib), ("production", B.build())):
        env = dict(os.environ, PACKINFER_LIB=path)
        f = str(tmp_path / f"{name}.pt")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "checked_run.py"), f], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "checked_run ok" in r.stdout, (name, r.stdout[-2000:], r.stderr[-2000:])
        assert "device check" not in r.stdout + r.stderr, (name, r.stdout[-2000:])
        outs[name] = torch.load(f)
    assert len(outs["checked"]) == len(outs["production"])
    for a, b in zip(outs["checked"], outs["production"]):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


@pytest.mark.gpu
def test_checked_build_traps_on_bad_row(tmp_path):
    """Negative control: with a row-table entry pointing past the end of Q, the checked library traps
    with its check message (the production library would read out of bounds)."""
    from paper_2602_06072_b200 import build as B
    lib = os.path.join(ROOT, "variants", "libpi_checks.so")
    if not os.path.exists(lib):
        B.build(True, False, lib, ("PI_CHECKS=1",))
    env = dict(os.environ, PACKINFER_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "checked_run.py"), str(tmp_path / "x.pt"),
                        "--corrupt"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, r.stdout[-2000:]
    assert "device check" in r.stdout + r.stderr, (r.stdout[-2000:], r.stderr[-2000:])
