"""CLI: profile (analytic) -> plan -> simulate on CPU, `run` on the B200."""
import json

import pytest

from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.cli import main


def _plan_files(tmp_path, model="tiny", b=2, stages=2, schedule="async", cap="16G"):
    g, p = tmp_path / "g.json", tmp_path / "p.json"
    assert main(["profile", model, "--micro-batch", str(b), "--analytic", "--out", str(g)]) == 0
    assert main(["plan", str(g), "--stages", str(stages), "--schedule", schedule,
                 "--capacity", cap, "--out", str(p)]) == 0
    return g, p


def test_cli_plan_and_simulate_match_library(tmp_path):
    g, p = _plan_files(tmp_path, "bert-base", 8, 4)
    graph = P.load_profile(str(g))
    plan = P.plan(graph, P.PlanConfig(stages=4, schedule=P.SCHEDULE_ASYNC, capacity=16 << 30,
                                      bandwidth=16 << 30))
    assert p.read_text() == P.plan_json(plan)
    out, trace = tmp_path / "r.json", tmp_path / "t.csv"
    assert main(["simulate", str(p), str(g), "--trace", str(trace), "--out", str(out)]) == 0
    rep = P.simulate(plan, graph, P.SimConfig(16, P.SCHEDULE_ASYNC, 16 << 30, 16 << 30))
    assert json.loads(out.read_text()) == json.loads(P.report_json(rep))
    assert trace.read_text() == P.trace_to_csv(rep)


def test_cli_exit_codes(tmp_path):
    g, _ = _plan_files(tmp_path)
    assert main(["plan", str(g), "--stages", "2", "--capacity", "1K"]) == 2  # infeasible
    assert main(["plan", str(g), "--stages", "2"]) == 1                      # usage
    assert main(["plan", str(tmp_path / "missing.json"), "--stages", "2", "--capacity", "1G"]) == 1
    assert main(["profile", "no-such-model", "--micro-batch", "1", "--analytic"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["async", "sync"])
def test_cli_run_reports_measured_trace(tmp_path, schedule):
    g, p = _plan_files(tmp_path, "tiny", 2, 2, schedule)
    out, trace = tmp_path / "r.json", tmp_path / "t.csv"
    assert main(["run", str(p), str(g), "--micro-batches", "4", "--steps", "2",
                 "--trace", str(trace), "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert len(doc["losses"]) == 4 and all(x > 0 for x in doc["losses"])
    assert doc["samples_per_s"] > 0 and doc["makespan_us"] > 0
    rows = trace.read_text().splitlines()
    assert rows[0] == "stage,mb,kind,start_us,end_us"
    assert len(rows) - 1 == doc["events"] == 2 * 2 * 4  # l stages x m micro-batches x {fwd, bwd}
