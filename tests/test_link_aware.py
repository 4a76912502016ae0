"""Link-aware eviction costs (beyond the reference, PlanConfig(link_aware=True)):
swaps share the host link, so once a stage's transfers exceed its compute time
recompute competes at its real price; the default stays bit-exact with
dawnplan (tests/test_planner_golden.py)."""
import json

from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.planner import memplan
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS


def _link_bytes(g, lo, hi, plan, bw):
    return sum(P.transfer_time_us(a.size, bw) for a in plan.actions if a.kind == "swap")


def test_link_aware_keeps_transfers_near_the_compute_budget():
    g = profile_graph(PRESETS["gpt2-xl"], 16)
    lo, hi, w, bw = 0, 56, 8, 48_000_000_000
    mp = g.segment_peak(lo, hi)
    cap = int(0.55 * w * mp)
    ref = memplan.optimize(g, lo, hi, micro_peak=mp, replica_weight=w, capacity=cap, bandwidth=bw)
    la = memplan.optimize_link_aware(g, lo, hi, micro_peak=mp, replica_weight=w, capacity=cap,
                                     bandwidth=bw)
    budget = g.segment_time(lo, hi)
    assert ref is not None and la is not None
    assert w * (mp - la.bytes_saved) <= cap
    # the reference plan overruns the link budget without charging it ...
    assert _link_bytes(g, lo, hi, ref, bw) > budget and ref.added_time < _link_bytes(g, lo, hi, ref, bw) - budget
    # ... the link-aware one charges every overflowing microsecond and uses recompute
    overflow = max(0, _link_bytes(g, lo, hi, la, bw) - budget)
    assert la.added_time >= overflow
    assert any(a.kind == "recompute" for a in la.actions)
    assert la.added_time <= ref.added_time + max(0, _link_bytes(g, lo, hi, ref, bw) - budget)


def test_link_aware_plan_roundtrips_and_default_doc_unchanged():
    g = profile_graph(PRESETS["tiny"], 2)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1, 1])
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, 2, P.SCHEDULE_ASYNC))
    base = dict(stages=2, schedule=P.SCHEDULE_ASYNC, capacity=int(0.6 * top), bandwidth=50 << 20)
    p0 = P.plan(g, P.PlanConfig(**base))
    assert "link_aware" not in json.loads(P.plan_json(p0))["config"]
    p1 = P.plan(g, P.PlanConfig(**base, link_aware=True))
    doc = json.loads(P.plan_json(p1))
    assert doc["config"]["link_aware"] is True
    assert P.plan_from_doc(g, doc).config.link_aware
