"""Max-trainable-batch harness (runtime/maxbatch.py): planning arms on CPU, the
on-GPU stage check (cap enforcement, no memory carried between trials) on a B200."""
import gc

import pytest
import torch

from paper_2505_05856_b200.kernels import release_workspaces
from paper_2505_05856_b200.runtime.maxbatch import GIB, check_stage, max_batch, try_batch
from paper_2505_05856_b200.runtime.model import PRESETS
from paper_2505_05856_b200.runtime.graph import profile_graph

BW = 48_000_000_000


@pytest.mark.parametrize("model", ["tiny", "tiny-t5"])
def test_planning_arms_cpu(model):
    cfg = PRESETS[model]
    cap = 2 * GIB
    best = {}
    for strat in ("even_compute", "even_compute_memopt", "dawnpiper"):
        b, hist = max_batch(cfg, 4, cap, BW, strat, b_max=256, run_gpu=False)
        assert b >= 1 and hist and hist[0]["b"] == 1
        feasible = [r["b"] for r in hist if r.get("feasible")]
        infeasible = [r["b"] for r in hist if not r.get("feasible")]
        assert max(feasible) == b
        assert all(x > b for x in infeasible)  # bisection brackets the answer
        best[strat] = b
    # memory optimisation never loses against the plain even-compute split
    assert best["even_compute_memopt"] >= best["even_compute"]
    assert best["dawnpiper"] >= best["even_compute"]


def test_try_batch_record_cpu():
    r = try_batch(PRESETS["tiny"], 4, 2, 2 * GIB, BW, "dawnpiper", run_gpu=False)
    assert r["feasible"] and len(r["cuts"]) == 1 and len(r["sched_peak_gib"]) == 2
    assert 0 < r["planner_capacity"] <= 2 * GIB - r["reserve"]


@pytest.mark.gpu
def test_check_stage_no_carryover_gpu():
    cfg = PRESETS["tiny"]
    b = 8
    g = profile_graph(cfg, b)
    r = try_batch(cfg, b, 2, 8 * GIB, BW, "even_compute", run_gpu=False)
    from paper_2505_05856_b200 import planner as P
    ample = P.PlanConfig(stages=2, schedule=P.SCHEDULE_ASYNC, capacity=1 << 62, bandwidth=BW)
    plan = P.plan_from_cuts(g, ample, r["cuts"])
    release_workspaces()  # scratch cached by earlier tests in this process
    gc.collect()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    peaks = []
    for _ in range(3):  # a fresh stream per trial: nothing may stay allocated afterwards
        c = check_stage(cfg, g, plan, 1, b, 8 * GIB)
        assert c.ok, c.error
        peaks.append(c.peak_bytes)
        assert torch.cuda.memory_allocated() == base
    assert peaks[0] == peaks[1] == peaks[2]


@pytest.mark.gpu
def test_check_stage_enforces_cap_gpu():
    cfg = PRESETS["tiny"]
    b = 8
    g = profile_graph(cfg, b)
    from paper_2505_05856_b200 import planner as P
    ample = P.PlanConfig(stages=2, schedule=P.SCHEDULE_ASYNC, capacity=1 << 62, bandwidth=BW)
    plan = P.plan_from_cuts(g, ample, P.compute_balanced(g, 0, len(g) - 1, [1, 1]).positions)
    c = check_stage(cfg, g, plan, 1, b, 1 << 20)  # 1 MiB: the weights alone do not fit
    assert not c.ok and "memory" in c.error.lower()


def test_release_workspaces_cpu():
    """The per-stream scratch cache drops its buffers (all, or one device's);
    torch.device / "cuda:k" / k name the same device key."""
    from paper_2505_05856_b200 import kernels as K
    K._WS.clear()
    K._WS[(0, 1234)] = torch.empty(1)
    K._WS[(1, 1234)] = torch.empty(1)
    K._WS[(1, 99)] = torch.empty(1)
    release_workspaces(torch.device("cuda", 0))
    assert sorted(K._WS) == [(1, 99), (1, 1234)]
    release_workspaces("cuda:1")
    assert not K._WS
    K._WS[(0, 5)] = torch.empty(1)
    release_workspaces()
    assert not K._WS


def test_host_bytes_match_executor_slots_cpu():
    """Pinned host bytes per stage = (l - x + 1) slots (1-based x, the ring depth
    StageExecutor allocates) of every swapped tensor."""
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.maxbatch import host_bytes
    cfg = PRESETS["tiny"]
    g = profile_graph(cfg, 8)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1] * 3)
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, 3, P.SCHEDULE_ASYNC))
    plan = P.plan(g, P.PlanConfig(stages=3, schedule=P.SCHEDULE_ASYNC, capacity=int(0.6 * top),
                                  bandwidth=16 << 30))
    hb = host_bytes(plan, 3)
    for x, m in enumerate(plan.memopt, start=1):
        swap = sum(a.size for a in m.actions if a.kind == "swap")
        assert hb[x - 1] == (3 - x + 1) * swap
    assert any(hb)
