"""Swap-engine knob sweep on the heaviest-memopt stage of a capped DawnPiper plan.

    python tools/memopt_knobs.py [--model gpt2-xl] [--b 16] [--cap-gib 40]

Prints one JSON line per (d2h_budget, prefetch_budget) setting with the
measured forward / backward / stall and the stage's device peak
(runtime/memprobe.py).
"""
import argparse, json, sys
sys.path.insert(0, ".")
from paper_2505_05856_b200.runtime.maxbatch import plan_for_cap
from paper_2505_05856_b200.runtime.memprobe import heaviest_stage, probe_stage
from paper_2505_05856_b200.runtime.model import PRESETS
from paper_2505_05856_b200.runtime.profiler import profile

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gpt2-xl")
ap.add_argument("--b", type=int, default=16)
ap.add_argument("--stages", type=int, default=8)
ap.add_argument("--cap-gib", type=float, default=40)
args = ap.parse_args()
cfg = PRESETS[args.model]
cap = int(args.cap_gib * (1 << 30))
g = profile(cfg, args.b, iters=5, warmup=2)
plan, pcfg = plan_for_cap(cfg, g, args.stages, cap, int(48e9), b=args.b)
x = heaviest_stage(plan)
MiB = 1 << 20
for d2h, pre in ((256 * MiB, 0), (1024 * MiB, 0), (256 * MiB, 2048 * MiB), (1024 * MiB, 2048 * MiB),
                 (2048 * MiB, 4096 * MiB)):
    r = probe_stage(cfg, g, plan, x, args.b, cap=cap,
                    swap_knobs={"d2h_budget": d2h, "prefetch_budget": pre})
    print(json.dumps({k: r[k] for k in ("stage", "swap_knobs", "fwd_us", "bwd_us", "added_time_us",
                                         "d2h", "h2d", "peak_bytes")}), flush=True)
