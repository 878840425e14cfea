"""Merge oracle — log-sum-exp combination of partial attention outputs, fp64.  TEST INFRASTRUCTURE.

The paper states only that split requests' "outputs [are] later merged in a lossless manner
consistent with FlashAttention semantics" and writes no equations (SPEC).
Reading R10: the standard streaming-softmax merge in natural-log units.
For partials (o_b, lse_b) of one query row over disjoint key segments:

    M   = max_b lse_b
    w_b = exp(lse_b - M)
    o   = sum_b w_b o_b / sum_b w_b
    lse = M + ln(sum_b w_b)

An empty partial is (0, -inf) and carries zero weight; if every partial is empty the result
is (0, -inf).
"""

from __future__ import annotations

import math
from typing import Sequence, Tuple

import numpy as np


def merge(partials: Sequence[Tuple[np.ndarray, float]]) -> Tuple[np.ndarray, float]:
    """Merge a list of (o [d], lse) partials of one row (the a9 equations)."""
    if not partials:
        raise ValueError("no partials")
    lses = [float(l) for _, l in partials]
    M = max(lses)
    d = np.asarray(partials[0][0]).shape[0]
    if M == -math.inf:
        return np.zeros(d), -math.inf
    w = [math.exp(l - M) for l in lses]
    W = math.fsum(w)
    o = np.zeros(d)
    for (ob, _), wb in zip(partials, w):
        o = o + wb * np.asarray(ob, dtype=np.float64)
    return o / W, M + math.log(W)


def merge2(a: Tuple[np.ndarray, float], b: Tuple[np.ndarray, float]):
    """Binary merge (used by the associativity pin)."""
    return merge([a, b])
