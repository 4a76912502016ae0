"""Compute- and memory-balanced cut positions (restates `dawnplan/balance.py`).

A cut position p puts canonical nodes <= p on the left; an l-way partition is
l-1 strictly increasing positions.

The reference computes the exact min-max compute split with an O(parts * n^2)
Fraction DP (balance.py:80-127), which is ~99% of its planning time (225 of
227 s at 290 nodes / 8 stages). Every caller on the plan
path passes unit weights, and for unit weights the same answer -- optimum value
and the lexicographically smallest optimal cut tuple -- follows from integer
arithmetic alone:

  * the optimum T* is the least integer T for which the range can be covered by
    at most `parts` segments of time <= T (times are non-negative ints, so T* is
    a segment sum and feasibility is monotone in T): binary search with an O(n)
    greedy check;
  * the reference's reconstruction takes, part by part, the smallest end e with
    seg(s, e) <= T* and an optimal-feasible suffix.  With equal weights a suffix
    starting at i can be split into exactly k non-empty parts of time <= T* iff
    minparts(i) <= k <= n - i, where minparts is the greedy segment count, which
    a two-pointer sweep gives for every i in O(n).

Non-unit weights keep an exact DP (integer cross-multiplied comparisons), used
only by tests and diagnostics.
"""

from __future__ import annotations

from dataclasses import dataclass
from bisect import bisect_left
from fractions import Fraction
from typing import Callable, List, Optional, Sequence, Tuple

from .profile import ComputationGraph

SCHEDULE_SYNC = "sync"
SCHEDULE_ASYNC = "async_1f1b"
SCHEDULES = (SCHEDULE_SYNC, SCHEDULE_ASYNC)


class InfeasibleCutError(ValueError):
    """A balance pass cannot produce the requested number of stages."""


@dataclass(frozen=True)
class Cut:
    """Strictly increasing cut positions (balance.py:34-46)."""

    positions: Tuple[int, ...]

    def __post_init__(self):
        ps = self.positions
        if any(b <= a for a, b in zip(ps, ps[1:])):
            raise ValueError(f"cut positions must be strictly increasing: {ps}")

    def __len__(self) -> int:
        return len(self.positions)


@dataclass(frozen=True)
class StageMemProfile:
    """Per-stage summary: one-micro-batch peak, residency-weighted peak, time."""

    stage: int
    micro_peak: int
    sched_peak: int
    time: int


def schedule_weight(schedule: str, stage: int, stages: int,
                    micro_batches: Optional[int] = None) -> int:
    """Residency multiplier (balance.py:65-77).

    Async 1F1B stage x keeps stages-x+1 micro-batches (and, in the B200 run,
    that many stashed weight versions) resident; sync keeps all m.
    """
    if schedule == SCHEDULE_ASYNC:
        return stages - stage + 1
    if schedule == SCHEDULE_SYNC:
        return micro_batches if micro_batches is not None else stages
    raise ValueError(f"unknown schedule {schedule!r}")


# -- exact min-max compute split ------------------------------------------------


def _check_split_args(lo: int, hi: int, weights: Sequence) -> Tuple[int, int, List[Fraction]]:
    parts = len(weights)
    n = hi - lo + 1
    if n <= 0:
        raise ValueError("empty node range")
    if parts < 1:
        raise ValueError("need at least one part")
    if parts > n:
        raise ValueError(f"{parts} parts exceed {n} nodes in range")
    w = [Fraction(x) for x in weights]
    if any(x <= 0 for x in w):
        raise ValueError("weights must be positive")
    return parts, n, w


def _unit_weight_split(times: List[int], parts: int) -> List[int]:
    """Offsets (relative to the range start) of the lexicographically smallest
    optimal min-max split of `times` into `parts` non-empty segments."""
    n = len(times)
    pre = [0]
    for t in times:
        pre.append(pre[-1] + t)

    def fits(cap: int) -> bool:
        used, run = 1, 0
        for t in times:
            if t > cap:
                return False
            if run + t > cap:
                used += 1
                run = t
                if used > parts:
                    return False
            else:
                run += t
        return True

    lo_t, hi_t = max(times), pre[-1]
    while lo_t < hi_t:
        mid = (lo_t + hi_t) // 2
        if fits(mid):
            hi_t = mid
        else:
            lo_t = mid + 1
    best = lo_t

    # minparts[i]: fewest segments of time <= best covering times[i:]
    minparts = [0] * (n + 1)
    j = n  # exclusive end of the greedy segment starting at i
    for i in range(n - 1, -1, -1):
        while pre[j] - pre[i] > best:
            j -= 1
        minparts[i] = 1 + minparts[j]

    cuts = []
    s = 0
    for p in range(parts - 1):
        tail = parts - p - 1
        for e in range(s, n - tail):
            if pre[e + 1] - pre[s] > best:
                break
            if minparts[e + 1] <= tail:
                cuts.append(e)
                s = e + 1
                break
        else:  # pragma: no cover - unreachable when best is optimal
            raise AssertionError("min-max reconstruction failed")
    return cuts


def _weighted_split(times: List[int], w: List[Fraction]) -> List[int]:
    """Exact suffix DP for arbitrary positive weights (same recurrence and
    tie-break as balance.py:99-126); loads compared by cross-multiplication."""
    parts, n = len(w), len(times)
    pre = [0]
    for t in times:
        pre.append(pre[-1] + t)

    def load(s: int, e: int, p: int) -> Fraction:
        return Fraction(pre[e + 1] - pre[s]) / w[p]

    INF = None
    best: List[List[Optional[Fraction]]] = [[INF] * (n + 1) for _ in range(parts)]
    for s in range(n):
        best[parts - 1][s] = load(s, n - 1, parts - 1)
    for p in range(parts - 2, -1, -1):
        tail = parts - p - 1
        nxt = best[p + 1]
        for s in range(n - tail - 1, -1, -1):
            acc = INF
            for e in range(s, n - tail):
                a = load(s, e, p)
                b = nxt[e + 1]
                v = a if (b is None or a >= b) else b
                if acc is None or v < acc:
                    acc = v
            best[p][s] = acc
    target = best[0][0]
    cuts = []
    s = 0
    for p in range(parts - 1):
        tail = parts - p - 1
        for e in range(s, n - tail):
            b = best[p + 1][e + 1]
            if load(s, e, p) <= target and b is not None and b <= target:
                cuts.append(e)
                s = e + 1
                break
    return cuts


def compute_balanced(g: ComputationGraph, lo: int, hi: int, weights: Sequence) -> Cut:
    """Exact min-max split of [lo, hi] into len(weights) weighted parts;
    lexicographically smallest optimal positions (balance.py:80-127)."""
    parts, n, w = _check_split_args(lo, hi, weights)
    times = [g.segment_time(k, k) for k in range(lo, hi + 1)]
    if parts == 1:
        return Cut(())
    if all(x == w[0] for x in w):
        offs = _unit_weight_split(times, parts)
    else:
        offs = _weighted_split(times, w)
    return Cut(tuple(lo + e for e in offs))


# -- memory balance ----------------------------------------------------------------


def _first_reach(g: ComputationGraph, start: int, hi: int, reached: Callable[[int], bool]) -> int:
    """Smallest k in [start, hi] whose running peak from `start` satisfies
    `reached`, or hi + 1.  The running peak of a segment grown to the right is
    non-decreasing (segment_peak is a range max), so this is a bisection over
    O(1) range-max queries instead of a node-by-node walk."""
    a, b = start, hi + 1
    while a < b:
        k = (a + b) // 2
        if reached(g.segment_peak(start, k)):
            b = k
        else:
            a = k + 1
    return a


def _crossing_walk(g: ComputationGraph, lo: int, hi: int, nbound: int,
                   target_of: Callable[[int], Fraction]) -> List[int]:
    """First-crossing cuts over [lo, hi]: a segment ends at the first node at
    which its running peak (from zero at the segment start) reaches the
    segment's target; at most nbound cuts."""
    cuts: List[int] = []
    start = lo
    while len(cuts) < nbound and start <= hi:
        target = Fraction(target_of(len(cuts)))
        num, den = target.numerator, target.denominator
        k = _first_reach(g, start, hi, lambda peak: peak * den >= num)
        if k > hi:
            break
        cuts.append(k)
        start = k + 1
    return cuts


def _halving_cut(g: ComputationGraph, lo: int, hi: int) -> int:
    """compute_balanced(g, lo, hi, [1, 1]).positions[0] by bisection over the
    time prefix sums: left time L(e) grows with e and right time R(e) shrinks,
    so max(L, R) is R until L >= R (from e*) and L after; the answer is the
    first e attaining the minimum."""
    pre = g._ptime
    base = pre[lo]
    total = pre[hi + 1] - base
    e_star = bisect_left(pre, base + (total + 1) // 2, lo + 1, hi + 1) - 1
    left_best = total - (pre[e_star] - base) if e_star > lo else None  # R(e* - 1)
    right_best = pre[e_star + 1] - base if e_star < hi else None      # L(e*)
    if right_best is None or (left_best is not None and left_best <= right_best):
        # first e with R(e) <= left_best, i.e. prefix index e + 1 reaching total - best
        return bisect_left(pre, base + total - left_best, lo + 1, e_star + 1) - 1
    return e_star


def _first_crossing(g: ComputationGraph, stages: int,
                    target_for: Callable[[int], Fraction]) -> Cut:
    n = len(g.nodes)
    if stages < 2:
        raise ValueError("need at least two stages")
    if stages > n:
        raise InfeasibleCutError(f"{stages} stages exceed {n} nodes")
    cuts = _crossing_walk(g, 0, n - 1, stages - 1, lambda j: target_for(j + 1))
    if len(cuts) < stages - 1:
        raise InfeasibleCutError(
            f"only {len(cuts) + 1} nonempty segments fit {stages} stage targets")
    if cuts[-1] >= n - 1:
        raise InfeasibleCutError("last stage would be empty")
    return Cut(tuple(cuts))


def memory_balanced_1f1b(g: ComputationGraph, stages: int) -> Cut:
    """Alg. 2 (balance.py:164-177): targets
    M_1 = peak / sum_i l/(l-i), M_x = l/(l-x+1) * M_1."""
    peak = g.peak_memory
    if peak <= 0:
        raise InfeasibleCutError("graph has no peak memory to balance")
    m1 = Fraction(peak) / sum(Fraction(stages, stages - i) for i in range(stages))
    return _first_crossing(g, stages, lambda x: Fraction(stages, stages - x + 1) * m1)


def memory_balanced_sync(g: ComputationGraph, stages: int) -> Cut:
    peak = g.peak_memory
    if peak <= 0:
        raise InfeasibleCutError("graph has no peak memory to balance")
    share = Fraction(peak, stages)
    return _first_crossing(g, stages, lambda x: share)


def split_pair(g: ComputationGraph, lo: int, hi: int, stages: int, schedule: str,
               left_stages: Sequence[int], right_stages: Sequence[int]) -> Tuple[int, int]:
    """(cb, mb) endpoints of the super-split search interval (balance.py:189-241)."""
    seq = list(left_stages) + list(right_stages)
    parts = len(seq)
    nl = len(left_stages)
    if parts == 2:
        cb = _halving_cut(g, lo, hi)
    else:
        cb = compute_balanced(g, lo, hi, [1] * parts).positions[nl - 1]

    if schedule == SCHEDULE_ASYNC:
        weights = [Fraction(1, stages - x + 1) for x in seq]
    elif schedule == SCHEDULE_SYNC:
        weights = [Fraction(1)] * parts
    else:
        raise ValueError(f"unknown schedule {schedule!r}")
    total = sum(weights)
    rpeak = Fraction(g.segment_peak(lo, hi))
    cuts = _crossing_walk(g, lo, hi, parts - 1, lambda j: rpeak * weights[j] / total)
    while len(cuts) < parts - 1:
        # targets never reached: pack the remaining boundaries against the tail
        nxt = hi - (parts - 1 - len(cuts))
        cuts.append(max(nxt, cuts[-1] + 1 if cuts else lo))
    mb = min(max(cuts[nl - 1], lo), hi - 1)
    return cb, mb


def stage_profiles(g: ComputationGraph, cut: Cut, stages: int, schedule: str,
                   micro_batches: Optional[int] = None) -> List[StageMemProfile]:
    if len(cut.positions) != stages - 1:
        raise ValueError("cut arity does not match stage count")
    bounds = [0, *[p + 1 for p in cut.positions], len(g.nodes)]
    out = []
    for x in range(1, stages + 1):
        lo, hi = bounds[x - 1], bounds[x] - 1
        micro = g.segment_peak(lo, hi)
        w = schedule_weight(schedule, x, stages, micro_batches)
        out.append(StageMemProfile(stage=x, micro_peak=micro, sched_peak=w * micro,
                                   time=g.segment_time(lo, hi)))
    return out
