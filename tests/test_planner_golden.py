"""Planner / schedule parity against the reference's own outputs.

tests/golden/planner_golden.json.gz was produced by oracle/gen_golden.py from the
unmodified reference (dawnplan 0.1.0): plan_json bytes (sha256 + parsed doc),
search traces, simulate() reports and trace CSV hashes, balance cuts.
"""
import hashlib
import json

import pytest

from paper_2505_05856_b200 import planner as P


def _cases(golden):
    for case in golden["cases"]:
        yield case, P.graph_from_doc(case["profile"])


def test_hash_and_doc_roundtrip(planner_golden):
    for case, g in _cases(planner_golden):
        assert P.canonical_hash(g) == case["hash"]
        assert P.profile_doc(g) == case["profile"]


def test_balance_cuts(planner_golden):
    for case, g in _cases(planner_golden):
        n = len(g)
        for bal in case["balance"]:
            s = bal["stages"]
            assert list(P.compute_balanced(g, 0, n - 1, [1] * s).positions) == bal["compute_balanced"]
            for name, fn in (("mem_1f1b", P.memory_balanced_1f1b), ("mem_sync", P.memory_balanced_sync)):
                want = bal[name]
                if isinstance(want, str):
                    with pytest.raises(P.InfeasibleCutError) as ei:
                        fn(g, s)
                    assert "ERR:" + str(ei.value) == want
                else:
                    assert list(fn(g, s).positions) == want
            got = P.split_pair(g, 0, n - 1, s, P.SCHEDULE_ASYNC, list(range(1, s // 2 + 1)),
                               list(range(s // 2 + 1, s + 1)))
            assert list(got) == bal["split_pair"]


def test_plans_byte_identical(planner_golden):
    checked = 0
    for case, g in _cases(planner_golden):
        for rec in case["plans"]:
            cfg = P.PlanConfig(stages=rec["stages"], schedule=rec["schedule"],
                               capacity=rec["capacity"], bandwidth=rec["bandwidth"])
            if "error" in rec:
                with pytest.raises(P.InfeasibleModelError) as ei:
                    P.plan(g, cfg)
                assert str(ei.value) == rec["error"]
                continue
            p, trace = P.plan_with_trace(g, cfg)
            pj = P.plan_json(p)
            assert hashlib.sha256(pj.encode()).hexdigest() == rec["plan_json_sha256"]
            assert json.loads(pj) == rec["plan_doc"]
            assert [[s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen] for s in trace] == rec["trace"]
            for sim in rec["sim"]:
                r = P.simulate(p, g, P.SimConfig(sim["m"], rec["schedule"], rec["bandwidth"], rec["capacity"]))
                rj = P.report_json(r)
                assert hashlib.sha256(rj.encode()).hexdigest() == sim["report_sha256"]
                assert hashlib.sha256(P.trace_to_csv(r).encode()).hexdigest() == sim["csv_sha256"]
            checked += 1
    assert checked > 300


def test_measured_baseline_profiles_plans_byte_identical():
    """Plans on the B200-measured BERT-base / BERT-large / GPT-2 XL / T5-large
    profiles (111-509 nodes, memopt-active capacities) against the unmodified
    reference's output (oracle/gen_golden_large.py)."""
    import gzip
    from pathlib import Path
    here = Path(__file__).parent / "golden"
    doc = json.loads(gzip.decompress((here / "planner_golden_large.json.gz").read_bytes()))
    graphs = {}
    big = 0
    for rec in doc["cases"]:
        name = rec["profile"]
        if name not in graphs:
            graphs[name] = P.graph_from_doc(json.loads(gzip.decompress(
                (here / "profiles" / f"{name}.json.gz").read_bytes())))
        g = graphs[name]
        assert P.canonical_hash(g) == rec["hash"]
        cfg = P.PlanConfig(stages=rec["stages"], schedule=rec["schedule"], capacity=rec["capacity"],
                           bandwidth=rec["bandwidth"])
        if "error" in rec:
            with pytest.raises(P.InfeasibleModelError) as ei:
                P.plan(g, cfg)
            assert str(ei.value) == rec["error"]
            continue
        p, trace = P.plan_with_trace(g, cfg)
        pj = P.plan_json(p)
        assert hashlib.sha256(pj.encode()).hexdigest() == rec["plan_json_sha256"], (name, rec["stages"])
        assert [[s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen] for s in trace] == rec["trace"]
        r = P.simulate(p, g, P.SimConfig(micro_batches=rec["sim"]["m"], schedule=rec["schedule"],
                                         bandwidth=rec["bandwidth"], capacity=rec["capacity"]))
        assert hashlib.sha256(P.report_json(r).encode()).hexdigest() == rec["sim"]["report_sha256"]
        big += len(g) >= 200 and any(m.actions for m in p.memopt)
    assert big >= 3
