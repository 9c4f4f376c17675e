"""Lanes whose PLCM orbit hits the guard set {0, p, 0.5} at a chosen stream
iteration, i.e. after the 256 exact warm-up steps (chaos.hpp:14), where the
GPU runs the speculative chain.  Test infrastructure.

With a dyadic p = 2^-s, the reference step x/p (chaos.cpp:28-32) is an exact
scaling by 2^s, so a seed x0 = m * 2^-E climbs exactly: x_k = m * 2^(sk - E).
E fixes the step at which the orbit reaches a guard value:
  m = 1: x_k = 0.5 (E = s*k + 1) or x_k = p (E = s*k + s);
  m = 3, p = 1/4: x_k = 0.75, and the next step folds to 0.25 = p and
  gives (p - p)/q = 0.
After a guard fires (chaos.cpp:15-24), p = 1/4 orbits fall back onto the
climb 2^-50, 2^-48, ... and hit p again every 25 iterations, so the guard
keeps firing in every later verify group and launch.

(1.0 is unreachable from a non-guard x: for x < 0.5, RN(x - p) misses q by at
least ulp(q), so (x - p)/q rounds below 1.)
"""
from __future__ import annotations

GUARD_EPS = 2.0 ** -52
WARMUP = 256


def step(x: float, p: float) -> float:
    """chaos.cpp:28-32 (no guard); Python floats are IEEE binary64."""
    if x > 0.5:
        x = 1.0 - x
    if x < p:
        return x / p
    return (x - p) / (0.5 - p)


def is_guard(x: float, p: float) -> bool:
    return x == 0.0 or x == p or x == 0.5 or x == 1.0


def guard(x: float, p: float) -> float:
    """chaos.cpp:15-24."""
    if is_guard(x, p):
        x += GUARD_EPS
        if x > 1.0:
            x -= 1.0
    return x


def stream_hits(x0: float, p: float, iterations: int) -> list[tuple[int, float]]:
    """(stream iteration, unguarded value) of every guard firing after the
    warm-up, following the reference generator (seed guard, warm-up)."""
    x = guard(x0, p)
    for _ in range(WARMUP):
        x = guard(step(x, p), p)
    hits = []
    for i in range(1, iterations + 1):
        y = step(x, p)
        if is_guard(y, p):
            hits.append((i, y))
        x = guard(y, p)
    return hits


def seed(kind: str, at: int, s: int = 2) -> tuple[float, float]:
    """(x0, p) whose stream iteration `at` (1-based) is a `kind` guard hit."""
    p = 2.0 ** -s
    k = WARMUP + at  # total steps from the seed to the hit
    if kind == "half":
        return 2.0 ** -(s * k + 1), p
    if kind == "p":
        return 2.0 ** -(s * k + s), p  # x_{k-1} = p*p, step k gives p
    if kind == "zero":
        assert s == 2
        return 3.0 * 2.0 ** -(2 * (k - 1) + 2), p  # x_{k-1} = 0.75
    raise ValueError(kind)


# (kind, stream iteration of the first hit, s): every seed is a normal double
CASES = [("half", 3, 2), ("half", 40, 2), ("half", 30, 3), ("p", 7, 2), ("p", 200, 2),
         ("zero", 60, 2), ("zero", 1, 2)]
