"""Host planner: bit-exact restatement of the reference `dawnplan` plan path.

Drop-in names (same signatures, results and errors as `dawnplan`):
profile model (`profile.py`), balance (`balance.py`), memopt (`memplan.py`),
BiPar search and plan files (`search.py`), schedule model (`schedule.py`).
"""

from .balance import (SCHEDULE_ASYNC, SCHEDULE_SYNC, SCHEDULES, Cut, InfeasibleCutError,
                      StageMemProfile, compute_balanced, memory_balanced_1f1b,
                      memory_balanced_sync, schedule_weight, split_pair, stage_profiles)
from .memplan import (MemOptAction, MemOptPlan, RecomputeCandidate, StageTimeline,
                      SwapCandidate, build_stage_timeline, collect_candidates,
                      exhaustive_optimize, optimize, producer_chain)
from .profile import (MIB, PROFILE_SCHEMA, ComputationGraph, ProfiledNode, ProfileParseError,
                      ProfileValidationError, TensorRef, canonical_hash, cumulative_series,
                      graph_from_doc, load_profile, memory_cdf, profile_doc, save_profile,
                      transfer_time_us)
from .schedule import (SimConfig, SimEvent, SimReport, async_iteration, async_ops,
                       boundary_bytes, boundary_producers, compare_plans, report_json,
                       simulate, sync_ops, trace_to_csv)
from .search import (CandidateCut, InfeasibleModelError, PartitionPlan, PlanConfig, SearchStep,
                     candidate_cuts, inevitable_comm, load_plan_doc, plan, plan_doc,
                     plan_from_cuts, plan_from_doc, plan_json, plan_with_trace, save_plan,
                     stage_bounds)
from .synth import gen_cnn_like, gen_transformer_like, gen_uniform
