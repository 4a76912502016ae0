"""Planner parity against the live reference, where it is mounted.

The committed goldens (test_planner_golden.py) pin the planner everywhere; in
the dev container the unmodified reference (`/root/reference/pkg/src`,
dawnplan 0.1.0) is also importable, and these tests compare this package's
search (`planner/search.py`: candidate walk, feasibility-first pair scan with
branch-and-bound) and eviction greedy (`planner/memplan.py`: presorted walk,
finisher heap) with it on freshly drawn cases.  They skip where the
reference is absent (e.g. the GPU box).
"""
import random
import tempfile
from pathlib import Path

import pytest

from paper_2505_05856_b200 import planner as P

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def R():
    import sys
    sys.path.insert(0, str(REF))
    import dawnplan
    return dawnplan


def _pair(R, rg):
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "g.json"
        R.save_profile(rg, f)
        return P.load_profile(f)


def _graphs(R):
    out = []
    for seed in range(1, 5):
        out.append(R.gen_transformer_like(2 + seed % 3, seed))
        out.append(R.gen_cnn_like(4 + 2 * seed, seed))
    return out


def test_optimize_matches_reference(R):
    from dawnplan import memopt as RM
    rng = random.Random(11)
    cases = 0
    for rg in _graphs(R):
        g = _pair(R, rg)
        n = len(g)
        for _ in range(120):
            lo = rng.randrange(n)
            hi = rng.randrange(lo, n)
            mp = g.segment_peak(lo, hi)
            w = rng.randint(1, 8)
            cap = max(1, int(w * mp * rng.uniform(0.05, 1.1)))
            bw = rng.choice([100 << 20, 1 << 30, 16 << 30])
            want = RM.optimize(rg, lo, hi, micro_peak=mp, replica_weight=w, capacity=cap, bandwidth=bw)
            got = P.optimize(g, lo, hi, micro_peak=mp, replica_weight=w, capacity=cap, bandwidth=bw)
            assert P.memplan.stage_feasible(g, lo, hi, micro_peak=mp, replica_weight=w,
                                            capacity=cap) == (want is not None)
            if want is None:
                assert got is None
                continue
            assert [(a.kind, a.tensor_id, a.size, a.overhead_us) for a in got.actions] == \
                [(a.kind, a.tensor_id, a.size, a.overhead_us) for a in want.actions]
            assert (got.bytes_saved, got.added_time) == (want.bytes_saved, want.added_time)
            cases += 1
    assert cases > 300


def test_split_pair_matches_reference(R):
    from paper_2505_05856_b200.planner import balance as B
    rng = random.Random(5)
    for rg in _graphs(R):
        g = _pair(R, rg)
        n = len(g)
        for _ in range(150):
            lo = rng.randrange(n - 1)
            hi = rng.randrange(lo + 1, n)
            assert B._halving_cut(g, lo, hi) == R.compute_balanced(rg, lo, hi, [1, 1]).positions[0]
            stages = rng.randint(2, 8)
            parts = rng.randint(2, min(stages, hi - lo + 1))
            first = rng.randint(1, stages - parts + 1)
            seq = list(range(first, first + parts))
            nl = rng.randint(1, parts - 1)
            for sched in (R.SCHEDULE_ASYNC, R.SCHEDULE_SYNC):
                assert tuple(P.split_pair(g, lo, hi, stages, sched, seq[:nl], seq[nl:])) == \
                    tuple(R.split_pair(rg, lo, hi, stages, sched, seq[:nl], seq[nl:]))


def test_plans_and_traces_match_reference(R):
    rng = random.Random(3)
    checked = 0
    for rg in _graphs(R):
        g = _pair(R, rg)
        n = len(g)
        for stages in (2, 3, 4, 8):
            if stages > n:
                continue
            for sched in (R.SCHEDULE_ASYNC, R.SCHEDULE_SYNC):
                cb = R.compute_balanced(rg, 0, n - 1, [1] * stages)
                top = max(p.sched_peak for p in R.stage_profiles(rg, cb, stages, sched))
                cap = max(1, int(rng.uniform(0.2, 1.05) * top))
                bw = rng.choice([100 << 20, 2 << 30, 16 << 30])
                cc = rng.choice([0.25, 0.5, 1.0])
                kw = dict(stages=stages, schedule=sched, capacity=cap, bandwidth=bw, comm_cap=cc)
                try:
                    rp, rt = R.plan_with_trace(rg, R.PlanConfig(**kw))
                except R.InfeasibleModelError as e:
                    with pytest.raises(P.InfeasibleModelError) as ei:
                        P.plan(g, P.PlanConfig(**kw))
                    assert str(ei.value) == str(e)
                    continue
                pp, pt = P.plan_with_trace(g, P.PlanConfig(**kw))
                assert P.plan_json(pp) == R.plan_json(rp)
                assert [(s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen) for s in pt] == \
                    [(s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen) for s in rt]
                checked += 1
    assert checked > 30
