"""Command-line front end: the reference's planner commands plus `profile` and `run`.

    python -m paper_2505_05856_b200 profile bert-large --micro-batch 8 --out g.json
    python -m paper_2505_05856_b200 plan g.json --stages 8 --capacity 40G --out p.json
    python -m paper_2505_05856_b200 simulate p.json g.json --micro-batches 32
    python -m paper_2505_05856_b200 run p.json g.json --micro-batches 32 --trace t.csv

`plan`, `simulate` and `compare` follow dawnplan's CLI (cli.py:78-125,
190-310): same arguments, same JSON on stdout (or --out), human summaries on
stderr, same exit codes (0 ok, 1 usage / input error, 2 infeasible model).
`run` is the B200 counterpart of `simulate`: it executes
the plan for real and writes the same report document (a superset: measured
losses, samples/s, device peak) and the same trace CSV (`trace_to_csv`,
simulate.py:86-90) from CUDA-event timings.  `profile` measures a model
preset's per-node B200 times into a schema-1 profile (`--analytic` writes the
structure with analytic times, no GPU needed).
"""

from __future__ import annotations

import argparse
import json
import re
import sys
from pathlib import Path
from typing import List, Optional

from . import planner as P

_SCHEDULES = {"sync": P.SCHEDULE_SYNC, "async": P.SCHEDULE_ASYNC}
_SIZE_RE = re.compile(r"^(\d+)([KMGT]?)$", re.IGNORECASE)
_SUFFIX = {"": 1, "K": 1024, "M": 1024 ** 2, "G": 1024 ** 3, "T": 1024 ** 4}


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise _UsageError(message)


def parse_size(text: str) -> int:
    """Bytes with optional K/M/G/T suffix (powers of 1024), as cli.py:47-52."""
    m = _SIZE_RE.match(text.strip())
    if not m:
        raise argparse.ArgumentTypeError(f"not a size: {text!r}")
    return int(m.group(1)) * _SUFFIX[m.group(2).upper()]


def _say(msg: str) -> None:
    print(msg, file=sys.stderr)


def _emit(text: str, out: Optional[str]) -> None:
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


def _build_parser() -> _Parser:
    p = _Parser(prog="dawnpiper-b200", description=__doc__)
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)

    f = sub.add_parser("profile", help="measure a model preset's per-node B200 profile")
    f.add_argument("model")
    f.add_argument("--micro-batch", type=int, required=True)
    f.add_argument("--iters", type=int, default=50)
    f.add_argument("--warmup", type=int, default=5)
    f.add_argument("--analytic", action="store_true", help="analytic node times (no GPU)")
    f.add_argument("--out")

    def planner_args(q):
        q.add_argument("profile")
        q.add_argument("--stages", type=int, required=True)
        q.add_argument("--schedule", choices=sorted(_SCHEDULES), default="async")
        q.add_argument("--capacity", type=parse_size, required=True)
        q.add_argument("--bandwidth", type=parse_size, default=16 * 1024 ** 3)
        q.add_argument("--comm-cap", type=float, default=0.5)
        q.add_argument("--out")

    q = sub.add_parser("plan", help="search for the min-bottleneck partition")
    planner_args(q)
    q.add_argument("--jobs", type=int, default=1)

    s = sub.add_parser("simulate", help="simulate a plan over its profile (analytic)")
    s.add_argument("plan")
    s.add_argument("profile")
    s.add_argument("--micro-batches", type=int, default=0)
    s.add_argument("--trace")
    s.add_argument("--out")

    r = sub.add_parser("run", help="execute a plan on B200s and report measured times")
    r.add_argument("plan")
    r.add_argument("profile")
    r.add_argument("--model", help="model preset (default: from the profile name)")
    r.add_argument("--micro-batch", type=int, default=0,
                   help="micro-batch size (default: from the profile name)")
    r.add_argument("--micro-batches", type=int, default=0,
                   help="0 picks the schedule default (l for sync, 4l for async)")
    r.add_argument("--steps", type=int, default=2, help="iterations; the last one is reported")
    r.add_argument("--devices", default="0", help="comma-separated CUDA device ids")
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--trace")
    r.add_argument("--out")
    r.add_argument("--static-peaks", action="store_true",
                   help="report static buffer bytes instead of measuring each stage's peak")

    c = sub.add_parser("compare", help="compute-balanced vs memory-balanced vs full planner")
    planner_args(c)
    c.add_argument("--micro-batches", type=int, default=0)
    c.add_argument("--jobs", type=int, default=1)
    return p


def _plan_config(args, jobs: int = 1) -> P.PlanConfig:
    return P.PlanConfig(stages=args.stages, schedule=_SCHEDULES[args.schedule],
                        capacity=args.capacity, bandwidth=args.bandwidth,
                        comm_cap=args.comm_cap, jobs=jobs)


def _default_m(stages: int, schedule: str, m: int) -> int:
    if m > 0:
        return m
    return stages if schedule == P.SCHEDULE_SYNC else 4 * stages


def _cmd_profile(args) -> int:
    from .runtime.model import PRESETS
    if args.model not in PRESETS:
        raise ValueError(f"unknown model {args.model!r}; presets: {sorted(PRESETS)}")
    if args.analytic:
        from .runtime.graph import profile_graph
        cfg = PRESETS[args.model]
        g = profile_graph(cfg, args.micro_batch, name=f"{cfg.name}_b{args.micro_batch}")
    else:
        from .runtime.profiler import profile
        g = profile(args.model, args.micro_batch, iters=args.iters, warmup=args.warmup)
    _emit(json.dumps(P.profile_doc(g), indent=2, sort_keys=True) + "\n", args.out)
    _say(f"{g.name}: {len(g)} nodes, total {g.segment_time(0, len(g) - 1) / 1000:.3f} ms, "
         f"peak {g.peak_memory / P.MIB:.1f} MiB")
    return 0


def _say_plan(p: P.PartitionPlan) -> None:
    cuts = ",".join(str(c) for c in p.cuts.positions)
    _say(f"{p.graph_name}: cuts [{cuts}], bottleneck {p.bottleneck_time / 1000:.3f} ms, "
         f"schedule {p.schedule}")
    for st, mo in zip(p.stages, p.memopt):
        acts = f", memopt {len(mo.actions)} actions +{mo.added_time} us" if mo.actions else ""
        _say(f"  stage {st.stage}: T {st.time / 1000:.3f} ms, "
             f"sched peak {st.sched_peak / P.MIB:.1f} MiB{acts}")


def _cmd_plan(args) -> int:
    g = P.load_profile(args.profile)
    p = P.plan(g, _plan_config(args, jobs=args.jobs))
    _emit(P.plan_json(p), args.out)
    _say_plan(p)
    return 0


def _load_plan(args):
    g = P.load_profile(args.profile)
    p = P.plan_from_doc(g, P.load_plan_doc(args.plan))
    return g, p


def _cmd_simulate(args) -> int:
    g, p = _load_plan(args)
    m = _default_m(p.config.stages, p.schedule, args.micro_batches)
    rep = P.simulate(p, g, P.SimConfig(micro_batches=m, schedule=p.schedule,
                                       bandwidth=p.config.bandwidth, capacity=p.config.capacity))
    _emit(P.report_json(rep), args.out)
    if args.trace:
        Path(args.trace).write_text(P.trace_to_csv(rep))
    _say(f"{g.name}: m={m}, iteration {rep.iteration_time / 1000:.3f} ms, "
         f"bubble {rep.bubble_ratio:.4f}, waste {rep.waste_ratio:.4f}")
    return 0


def _model_of(args, g):
    from .runtime.model import PRESETS
    name, b = args.model, args.micro_batch
    base, _, bs = g.name.rpartition("_b")
    if not name:
        name = base
    if b <= 0:
        if not bs.isdigit():
            raise ValueError(f"cannot infer the micro-batch size from {g.name!r}; pass --micro-batch")
        b = int(bs)
    if name not in PRESETS:
        raise ValueError(f"cannot infer the model of {g.name!r}; pass --model")
    return PRESETS[name], b


def _cmd_run(args) -> int:
    from .runtime.pipeline import RunConfig, run
    g, p = _load_plan(args)
    model, b = _model_of(args, g)
    m = _default_m(p.config.stages, p.schedule, args.micro_batches)
    devices = tuple(int(d) for d in args.devices.split(",") if d.strip())
    cfg = RunConfig(micro_batches=m, micro_batch_size=b, devices=devices, seed=args.seed,
                    trace=True, capacity=p.config.capacity,
                    measure_stage_peaks=not args.static_peaks)
    try:
        rep = run(p, g, cfg, model=model, steps=max(1, args.steps))
    except Exception as e:  # OOM under the cap = the plan does not fit this device
        if "out of memory" in str(e).lower():
            raise P.InfeasibleModelError(f"run exceeded the {p.config.capacity}-byte cap: {e}")
        raise
    _emit(json.dumps(rep.to_doc(), indent=2, sort_keys=True) + "\n", args.out)
    if args.trace:
        Path(args.trace).write_text(P.trace_to_csv(rep))
    _say(f"{g.name}: m={m}, measured iteration {rep.iteration_time / 1000:.3f} ms, "
         f"{rep.samples_per_s:.1f} samples/s, bubble {rep.bubble_ratio:.4f}")
    return 0


def _cmd_compare(args) -> int:
    g = P.load_profile(args.profile)
    n = len(g)
    cfg = _plan_config(args, jobs=args.jobs)
    m = _default_m(cfg.stages, cfg.schedule, args.micro_batches)
    sim_cfg = P.SimConfig(micro_batches=m, schedule=cfg.schedule, bandwidth=cfg.bandwidth,
                          capacity=cfg.capacity)
    cb = P.compute_balanced(g, 0, n - 1, [1] * cfg.stages)
    mb = (P.memory_balanced_sync(g, cfg.stages) if cfg.schedule == P.SCHEDULE_SYNC
          else P.memory_balanced_1f1b(g, cfg.stages))
    rows = []
    for label, p in (
            ("compute_balanced", P.plan_from_cuts(g, cfg, cb.positions, require_feasible=False)),
            ("memory_balanced", P.plan_from_cuts(g, cfg, mb.positions, require_feasible=False)),
            ("planner", P.plan(g, cfg))):
        r = P.simulate(p, g, sim_cfg)
        rows.append({"strategy": label, "cuts": list(p.cuts.positions),
                     "bottleneck_us": p.bottleneck_time, "iteration_time_us": r.iteration_time,
                     "bubble_ratio": r.bubble_ratio, "waste_ratio": r.waste_ratio,
                     "per_stage_peak_bytes": list(r.per_stage_peak),
                     "capacity_exceeded_stages": list(r.capacity_exceeded)})
    _emit(json.dumps({"micro_batches": m, "rows": rows}, indent=2, sort_keys=True) + "\n", args.out)
    _say(f"{g.name}: schedule {cfg.schedule}, m={m}")
    return 0


_COMMANDS = {"profile": _cmd_profile, "plan": _cmd_plan, "simulate": _cmd_simulate,
             "run": _cmd_run, "compare": _cmd_compare}


def main(argv: Optional[List[str]] = None) -> int:
    parser = _build_parser()
    try:
        args = parser.parse_args(argv)
    except _UsageError:
        return 1
    except SystemExit as e:  # --help
        return int(e.code or 0)
    try:
        return _COMMANDS[args.command](args)
    except (P.InfeasibleModelError, P.InfeasibleCutError) as e:
        _say(f"infeasible: {e}")
        return 2
    except (P.ProfileParseError, P.ProfileValidationError) as e:
        _say(f"invalid profile: {e}")
        return 1
    except (ValueError, OSError) as e:
        _say(f"error: {e}")
        return 1


if __name__ == "__main__":
    sys.exit(main())
