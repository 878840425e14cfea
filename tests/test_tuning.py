"""Adaptive capacity policy (NEXT-2): offline sweep picks the cheapest C, the online
tuner converges to the optimum within a few dozen steps from per-step samples, and follows a
workload shift (CPU only: the costs are synthetic convex curves with deterministic noise)."""

import math

import pytest

from paper_2602_06072_b200.tuning import CapacityTuner, offline_profile

CANDS = [1024, 2048, 4096, 8192, 16384]


def convex(opt):
    # convex in log2(C) with its minimum at `opt` (the paper reports a convex trend)
    return lambda c: 1.0 + 0.3 * (math.log2(c) - math.log2(opt)) ** 2


def test_offline_profile_picks_minimum():
    f = convex(2048)
    prof = offline_profile(f, CANDS)
    assert min(prof, key=prof.get) == 2048
    assert set(prof) == set(CANDS)


@pytest.mark.parametrize("opt", CANDS)
def test_online_converges(opt):
    f = convex(opt)
    tu = CapacityTuner(CANDS)
    picks = []
    for k in range(40):
        c = tu.choose()
        noise = 0.01 * ((k * 7919) % 13 - 6) / 6.0          # deterministic +-1 %
        tu.observe(c, f(c) * (1 + noise))
        picks.append(c)
    assert tu.best() == opt
    # after warm-up, at least 3/4 of the choices exploit the optimum
    tail = picks[len(CANDS):]
    assert sum(p == opt for p in tail) >= 0.75 * len(tail)


def test_online_follows_shift_and_uses_prior():
    prior = offline_profile(convex(8192), CANDS)
    tu = CapacityTuner(CANDS, prior=prior)
    assert tu.choose() == 8192                                # the prior's best, no warm-up
    f = convex(2048)                                          # workload shift: optimum moves
    for _ in range(60):
        c = tu.choose()
        tu.observe(c, f(c))
    assert tu.best() == 2048


def test_rejects_unknown_capacity():
    tu = CapacityTuner(CANDS)
    with pytest.raises(ValueError):
        tu.observe(3000, 1.0)
    with pytest.raises(ValueError):
        CapacityTuner([])
