"""Adaptive group capacity C (NEXT-2; PackInfer §3.1 "Adaptive Grouping").

The paper picks C by offline profiling over a range of group sizes and refines it online from
per-step latency samples ("each decoding step naturally yields one performance sample").  This
module is that policy, host-side and deterministic; the measurements come from the caller (CUDA
events around the hot path, scripts/c_sweep.py for the offline sweep on B200).  A change of C
takes effect at the next consolidation (a regroup, Eq. 4), so `CapacityTuner.choose` is meant to
be called when the caller re-plans with relayout.
"""

from __future__ import annotations

from typing import Callable, Dict, Iterable, List, Optional, Sequence


def offline_profile(measure: Callable[[int], float], candidates: Iterable[int], reps: int = 3) -> Dict[int, float]:
    """Offline sweep: median of `reps` calls of measure(C) (cost per unit of work, lower
    is better) for every candidate C.  Returns {C: cost}."""
    out = {}
    for c in candidates:
        xs = sorted(float(measure(int(c))) for _ in range(reps))
        out[int(c)] = xs[len(xs) // 2]
    return out


class CapacityTuner:
    """Online refinement of C from per-step samples.

    State per candidate: an exponentially weighted mean of the observed cost (per unit of work,
    e.g. ms per KV token) with decay `decay`, so that a workload shift is tracked.  Policy:
      1. warm-up: every candidate without a sample is tried once, in the order of the offline
         prior (best first) when one is given, else in the given order;
      2. exploit: the candidate with the lowest mean;
      3. every `probe_every` choices, probe the untried-longest neighbour (in sorted C order) of
         the current best, so a moved optimum is found within a few dozen steps.
    Deterministic: no random numbers."""

    def __init__(self, candidates: Sequence[int], prior: Optional[Dict[int, float]] = None,
                 decay: float = 0.7, probe_every: int = 8):
        if not candidates:
            raise ValueError("no candidates")
        self.cands: List[int] = sorted(int(c) for c in set(candidates))
        self.decay = float(decay)
        self.probe_every = int(probe_every)
        self.mean: Dict[int, Optional[float]] = {c: None for c in self.cands}
        self.last_seen: Dict[int, int] = {c: -1 for c in self.cands}
        self.t = 0
        order = list(self.cands)
        if prior:
            for c, v in prior.items():
                if int(c) in self.mean:
                    self.mean[int(c)] = float(v)
            order = sorted(self.cands, key=lambda c: (prior.get(c, float("inf")), c))
        self._warm = [c for c in order if self.mean[c] is None]

    def best(self) -> int:
        known = [c for c in self.cands if self.mean[c] is not None]
        if not known:
            return self.cands[0]
        return min(known, key=lambda c: (self.mean[c], c))

    def choose(self) -> int:
        self.t += 1
        if self._warm:
            return self._warm[0]
        b = self.best()
        if self.probe_every > 0 and self.t % self.probe_every == 0:
            i = self.cands.index(b)
            nb = [self.cands[j] for j in (i - 1, i + 1) if 0 <= j < len(self.cands)]
            if nb:
                return min(nb, key=lambda c: (self.last_seen[c], c))
        return b

    def observe(self, c: int, cost: float) -> None:
        c = int(c)
        if c not in self.mean:
            raise ValueError(f"unknown capacity {c}")
        m = self.mean[c]
        self.mean[c] = float(cost) if m is None else self.decay * m + (1.0 - self.decay) * float(cost)
        self.last_seen[c] = self.t
        if self._warm and self._warm[0] == c:
            self._warm.pop(0)
        elif c in self._warm:
            self._warm.remove(c)
