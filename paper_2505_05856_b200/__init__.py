"""B200-native DawnPiper pipeline-training step (drop-in for the dawnplan path).

  g = profile(model, micro_batch)         -> ComputationGraph (schema-1, measured on B200)
  p = plan(g, PlanConfig(...))            -> PartitionPlan    (bit-exact with dawnplan)
  r = run(p, g, RunConfig(...))           -> RunReport        (real 1F1B run; SimReport superset)

The planner names are re-exported here exactly as dawnplan exports them.
"""
from .planner import *  # noqa: F401,F403
from .planner import __dict__ as _pd  # noqa: F401


def run(*args, **kwargs):
    from .runtime.pipeline import run as _run
    return _run(*args, **kwargs)


def profile(*args, **kwargs):
    from .runtime.profiler import profile as _profile
    return _profile(*args, **kwargs)
