"""Training-step parity at the BASELINE configurations' real widths.

The toy-size parity tests (test_pipeline_gpu.py) cover the schedule and
executor logic; these run the kernels at the shapes the bench runs them --
head dims, head counts, vocabularies (and their 64-padding), sequence lengths
-- against the CPU fp32 oracle (oracle/train_ref.py) on the same seeded
inputs and init:

* C1 (BASELINE.md's CPU-baseline / parity configuration): BERT-base, 12
  layers, s128, a 4-stage DawnPiper plan built from the B200-measured profile,
  async 1F1B in `_async_ops` order (simulate.py:211-222), b=8, m=16, seed 0.
* Full-width slices (2 layers each) of BERT-large (H1024, 16 heads, s512,
  V30522), GPT-2 XL (H1600, 25 heads, causal s1024, V50257 padded to 50304)
  and T5-large (d1024, 16 heads, src 512 / tgt 128 cross-attention,
  V32128), each partitioned by the planner under a capacity and link
  bandwidth at which its plan contains both swap and recompute actions, so
  the swap engine and recompute replay run at real sizes.

Tolerance (BASELINE.json north_star, bf16): per-micro-batch losses within
rel 2e-2; every parameter within rel 2e-2 (Frobenius) and its update
direction within cosine 0.95 (see test_pipeline_gpu._compare).  The AdamW
learning rate is 1e-4 (BERT pre-training's): with PipeDream's update after
every micro-batch, m = 16 steps at 1e-3 move the small-gradient key
projections of the deep layers by as much as their init, and Adam's
normalised steps turn bf16 rounding of those near-zero gradients into
+-lr sign flips (measured: b8-b11 qkv.weight rel 2.2-3.5% at update cosine
0.989-0.996), which would test Adam's noise amplification, not the step.
"""
import dataclasses

import pytest

from test_pipeline_gpu import _compare

pytestmark = pytest.mark.gpu


def _memopt_plan(cfg, b, stages):
    """A DawnPiper plan of `cfg` whose memopt has both swaps and recomputes:
    the smallest capacity fraction / link bandwidth pair (scanned in order)
    at which the planner mixes both kinds."""
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    g = profile_graph(cfg, b)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1] * stages)
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, stages, P.SCHEDULE_ASYNC))
    for bw in (16 << 30, 256 << 20):
        for frac in [x / 100 for x in range(90, 25, -5)]:
            pc = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=int(frac * top),
                              bandwidth=bw)
            try:
                plan = P.plan(g, pc)
            except P.InfeasibleModelError:
                continue
            kinds = {a.kind for m in plan.memopt for a in m.actions}
            if kinds == {"swap", "recompute"}:
                return g, plan
    raise AssertionError(f"{cfg.name}: no plan with both swap and recompute actions")


def test_c1_bert_base_measured_profile_four_stages():
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.model import PRESETS
    from paper_2505_05856_b200.runtime.profiler import profile
    cfg = PRESETS["bert-base"]
    g = profile(cfg, 8, iters=5, warmup=2)  # measured B200 node times
    assert len(g) == 12 * 9 + 3
    plan = P.plan(g, P.PlanConfig(stages=4, schedule=P.SCHEDULE_ASYNC, capacity=40 << 30,
                                  bandwidth=16 << 30))
    _compare(cfg, g, plan, b=8, m=16, steps=1, seed=0, lr=1e-4)


def _slice(name, **kw):
    from paper_2505_05856_b200.runtime.model import PRESETS
    base = PRESETS[name]
    return dataclasses.replace(base, name=f"{name}-slice", **kw)


def test_bert_large_slice_swap_and_recompute():
    cfg = _slice("bert-large", layers=2)
    g, plan = _memopt_plan(cfg, 4, 2)
    _compare(cfg, g, plan, b=4, m=4, steps=1, seed=0, lr=1e-4)


def test_gpt2_xl_slice_swap_and_recompute():
    cfg = _slice("gpt2-xl", layers=2)
    assert cfg.vocab_padded == 50304 and cfg.head_dim == 64 and cfg.causal
    g, plan = _memopt_plan(cfg, 1, 2)
    _compare(cfg, g, plan, b=1, m=4, steps=1, seed=0, lr=1e-4)


def test_t5_large_slice_swap_and_recompute():
    cfg = _slice("t5-large", layers=2, dec_layers=2)
    assert (cfg.seq, cfg.tgt_seq) == (512, 128)
    g, plan = _memopt_plan(cfg, 4, 2)
    _compare(cfg, g, plan, b=4, m=4, steps=1, seed=0, lr=1e-4)


def test_bert_large_full_depth_bench_plan():
    """The bench's configuration at full depth: BERT-large 24 layers, s512, the
    8-stage DawnPiper plan from the B200-measured profile, co-located stages on
    concurrent streams with zero-copy hand-off (b=2, m=8 to bound CPU time)."""
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.model import PRESETS
    from paper_2505_05856_b200.runtime.profiler import profile
    cfg = PRESETS["bert-large"]
    g = profile(cfg, 2, iters=3, warmup=2)
    plan = P.plan(g, P.PlanConfig(stages=8, schedule=P.SCHEDULE_ASYNC, capacity=160 << 30,
                                  bandwidth=64 << 30))
    _compare(cfg, g, plan, b=2, m=8, steps=1, seed=0, lr=1e-4)


def test_gpt2_xl_full_depth_memopt_plan():
    """GPT-2 XL, 48 layers, s1024, 8 stages under a capacity at half the
    compute-balanced split's largest stage, so the plan swaps and recomputes
    across the whole depth (b=1, m=2)."""
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    from paper_2505_05856_b200.runtime.model import PRESETS
    cfg = PRESETS["gpt2-xl"]
    g = profile_graph(cfg, 1)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1] * 8)
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, 8, P.SCHEDULE_ASYNC))
    plan = P.plan(g, P.PlanConfig(stages=8, schedule=P.SCHEDULE_ASYNC, capacity=top // 2,
                                  bandwidth=16 << 30))
    assert sum(len(m.actions) for m in plan.memopt) > 50
    _compare(cfg, g, plan, b=1, m=2, steps=1, seed=0, lr=1e-4)
