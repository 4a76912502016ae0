"""Known-answer tests the reference suite pins.

Each value below is quoted from the reference tests (file:line in comments),
replayed against this package's planner and schedule model.
"""
import pytest

from paper_2505_05856_b200 import planner as P

MIB = 1 << 20
GIB = 1 << 30
BW16 = 16 * GIB
BW100M = 100 * MIB


def chain(name, times, mems, fwd_times=None, params=None, releases=None,
          saved_sizes=None, saved_access=None):
    n = len(times)
    nodes = []
    for i in range(n):
        nid = f"n{i}"
        t_f = fwd_times[i] if fwd_times is not None else times[i] // 2
        saved = ()
        if saved_sizes is not None and saved_sizes[i] > 0:
            acc = saved_access[i] if saved_access is not None else i
            saved = (P.TensorRef(f"{nid}.a", saved_sizes[i], nid, acc),)
        nodes.append(P.ProfiledNode(
            id=nid, depth=i, fwd_start=i, t_f=t_f, t_b=times[i] - t_f, m_a=mems[i],
            m_p=params[i] if params else 0, m_d=releases[i] if releases else 0,
            saved=saved, consumers=(f"n{i + 1}",) if i + 1 < n else ()))
    return P.ComputationGraph.build(name, nodes)


def saved_chain(times, mems):
    return chain("sc", times, mems, saved_sizes=list(mems))


def acfg(stages=2, capacity=12 * MIB, bandwidth=BW16):
    return P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=capacity, bandwidth=bandwidth)


def test_memory_balanced_fixtures(uni8, tri4):
    # test_acceptance.py:85-99
    cu = P.memory_balanced_1f1b(uni8, 2)
    ct = P.memory_balanced_1f1b(tri4, 2)
    assert cu.positions == (2,)
    assert tuple(p.sched_peak for p in P.stage_profiles(uni8, cu, 2, P.SCHEDULE_ASYNC)) == (6 * MIB, 5 * MIB)
    assert ct.positions == (0,)
    assert tuple(p.sched_peak for p in P.stage_profiles(tri4, ct, 2, P.SCHEDULE_ASYNC)) == (8 * MIB, 6 * MIB)


def test_compute_balanced_fixtures(uni8, tri4):
    # test_balance.py:63-74
    assert P.compute_balanced(uni8, 0, 7, [1, 1]).positions == (3,)
    assert P.compute_balanced(uni8, 0, 7, [1] * 4).positions == (1, 3, 5)
    assert P.compute_balanced(tri4, 0, 3, [1, 1]).positions == (2,)
    assert P.compute_balanced(tri4, 0, 3, [1, 2]).positions == (1,)
    assert P.compute_balanced(uni8, 2, 7, [1, 1]).positions == (4,)
    with pytest.raises(ValueError):
        P.compute_balanced(tri4, 0, 3, [1] * 5)
    with pytest.raises(ValueError, match="positive"):
        P.compute_balanced(uni8, 0, 7, [1, 0])


def test_compute_balanced_matches_brute_force():
    import itertools
    import random
    rnd = random.Random(7)
    for _ in range(150):
        n = rnd.randint(2, 9)
        times = [rnd.choice([0, 1, 3, 10, 50, 100]) for _ in range(n)]
        g = chain("bf", [2 * t for t in times], [MIB] * n)
        parts = rnd.randint(1, n)
        weights = [rnd.choice([1, 1, 2, 3]) for _ in range(parts)] if rnd.random() < 0.4 else [1] * parts
        best = None
        for cuts in itertools.combinations(range(n - 1), parts - 1):
            b = [0, *[c + 1 for c in cuts], n]
            from fractions import Fraction
            v = max(Fraction(g.segment_time(b[i], b[i + 1] - 1), weights[i]) for i in range(parts))
            if best is None or v < best[0]:
                best = (v, cuts)
        assert P.compute_balanced(g, 0, n - 1, weights).positions == best[1]


def test_planner_kats(uni8, tri4):
    # test_partition.py:136-183
    p = P.plan(uni8, acfg(capacity=12 * MIB))
    assert p.cuts.positions == (3,) and p.bottleneck_time == 4000
    p = P.plan(uni8, acfg(capacity=7 * MIB))
    assert p.cuts.positions == (2,) and p.effective_times() == (3000, 5000)
    p = P.plan(uni8, acfg(stages=4, capacity=12 * MIB))
    assert p.cuts.positions == (1, 3, 5)
    with pytest.raises(P.InfeasibleModelError,
                       match=r"stage 1 of the compute-balanced baseline needs 8388608 bytes"):
        P.plan(uni8, acfg(capacity=2 * MIB))
    g = P.gen_uniform(8, 1000, MIB)
    p = P.plan(g, acfg(capacity=2 * MIB))
    assert p.cuts.positions == (3,) and [len(m.actions) for m in p.memopt] == [3, 2]
    p, trace = P.plan_with_trace(tri4, acfg(capacity=9 * MIB))
    assert p.cuts.positions == (0,) and p.bottleneck_time == 9000
    assert [(s.lo, s.hi, s.cb, s.mb, s.chosen) for s in trace] == [(0, 3, 2, 0, 0)]


def test_memopt_kats():
    # test_memopt.py:22-26,110-160
    g = saved_chain([1000] * 8, [MIB] * 8)
    tl = P.build_stage_timeline(g, 0, 3)
    assert tl.fwd_end == (500, 1000, 1500, 2000) and tl.bwd_start == (3500, 3000, 2500, 2000)
    g = saved_chain([100] * 4, [MIB] * 4)
    plan = P.optimize(g, 0, 3, micro_peak=4 * MIB, replica_weight=1, capacity=MIB, bandwidth=BW100M)
    assert [(a.kind, a.tensor_id, a.overhead_us) for a in plan.actions] == [
        ("recompute", "n0.a", 50), ("recompute", "n2.a", 50), ("swap", "n3.a", 20000)]
    assert plan.added_time == 20100
    sizes = [MIB, MIB, MIB, 4 * MIB]
    g = chain("fin", [100] * 4, sizes, fwd_times=[0] * 4, saved_sizes=sizes)
    plan = P.optimize(g, 0, 3, micro_peak=7 * MIB, replica_weight=1, capacity=int(2.5 * MIB), bandwidth=BW100M)
    assert [(a.kind, a.tensor_id, a.overhead_us) for a in plan.actions] == [
        ("swap", "n0.a", 19700), ("swap", "n3.a", 80000)]
    g = saved_chain([100] * 2, [MIB] * 2)
    plan = P.optimize(g, 0, 1, micro_peak=2 * MIB, replica_weight=1, capacity=2 * MIB - 1,
                      bandwidth=13_981_013_334)
    assert len(plan.actions) == 1 and plan.actions[0].kind == "swap"


def _sim(g, stages, cuts, m, sched=P.SCHEDULE_ASYNC, capacity=GIB):
    p = P.plan_from_cuts(g, P.PlanConfig(stages, sched, capacity, BW16), cuts)
    return P.simulate(p, g, P.SimConfig(m, sched, BW16, capacity))


def test_schedule_kats(uni8):
    # test_simulate.py:61-68,102-137,216-223
    g = P.gen_uniform(8, 2000, 0)
    r = _sim(g, 4, [1, 3, 5], 4, P.SCHEDULE_SYNC)
    assert r.makespan == 28000 and r.bubble_ratio == pytest.approx(3 / 7, abs=1e-12)
    r = _sim(g, 4, [1, 3, 5], 4)
    assert [sum(1 for e in r.trace if e.stage == x and e.phase == "warmup") for x in (1, 2, 3, 4)] == [3, 2, 1, 0]
    r = _sim(g, 4, [1, 3, 5], 2)
    assert [sum(1 for e in r.trace if e.stage == x and e.phase == "warmup") for x in (1, 2, 3, 4)] == [2, 2, 1, 0]
    assert _sim(g, 4, [1, 3, 5], 16).iteration_time == 4000.0
    assert _sim(g, 8, list(range(7)), 16).iteration_time == 2000.0
    r = _sim(uni8, 2, [2], 1, capacity=12 * MIB)
    assert r.iteration_time == float(r.makespan) == 8124.0
    comm = [e for e in r.trace if e.kind == "comm"]
    assert (comm[0].stage, comm[0].mb, comm[0].start, comm[0].end) == (1, 1, 1500, 1562)


def test_async_ops_order():
    # l=4, m=8, x=1
    ops = [f"{k[0].upper()}{j}" for k, j, _ in P.async_ops(4, 8, 1)]
    assert ops == "F1 F2 F3 F4 B1 F5 B2 F6 B3 F7 B4 F8 B5 B6 B7 B8".split()


def test_skew9_appendix_a():
    # test_acceptance.py:168-187 (Appendix A): effective times and ratio 1.9623
    times = [29104, 47786, 30000, 29914, 53850, 53851, 2385, 138000, 145890]
    mems = [6 * MIB, 16 * MIB, 64 * 1024, 2 * MIB, 4 * MIB, 4 * MIB, 64 * 1024, 64 * 1024, 8 * MIB]
    fwd = [t // 2 for t in times]
    fwd[1] = 30000
    g = chain("skew9", times, mems, fwd_times=fwd, saved_sizes=list(mems[:8]) + [0],
              saved_access=[i + 1 for i in range(9)])
    cfg = P.PlanConfig(4, P.SCHEDULE_ASYNC, 64 * MIB, 100 * MIB)
    pa = P.plan_from_cuts(g, cfg, (0, 3, 5))
    pb = P.plan_from_cuts(g, cfg, (2, 6, 7))
    assert pa.effective_times() == (29104, 107700, 107701, 286275)
    assert pb.effective_times() == (136890, 140000, 138000, 145890)
    assert [(a.kind, a.tensor_id) for m in pb.memopt for a in m.actions] == [("recompute", "n1.a")]
    ra, rb, ratio = P.compare_plans(pa, pb, g, P.SimConfig(16, P.SCHEDULE_ASYNC, 100 * MIB, 64 * MIB))
    assert ratio == pytest.approx(1.9623, abs=1e-4)
    assert not ra.capacity_exceeded and not rb.capacity_exceeded
