"""Max trainable micro-batch under a per-GPU cap: DawnPiper plan vs even-compute split.

    python tools/max_batch.py [--model gpt2-xl] [--stages 8] [--cap-gib 40] [--calibrate]
                              [--no-gpu] [--no-timing] [--out FILE]

For each strategy (even-compute split, even-compute split + the same memopt
policy, DawnPiper) the largest micro-batch whose plan fits the cap -- every
stage run on the B200 under the cap (runtime/maxbatch.py) -- and, at that
micro-batch, every stage timed alone under the cap (runtime/memprobe.py) with
the 1F1B throughput those stage times give on l GPUs.

--calibrate first measures the optimizer / gradient-buffer / workspace bytes
the planner's model leaves out (maxbatch.calibrate_overhead: every stage of the
even split at b = 1, 2) instead of using the round-1 hand calibration.
"""
import argparse, json, sys, time
sys.path.insert(0, ".")
from paper_2505_05856_b200.runtime.maxbatch import (DEFAULT_OVERHEAD, calibrate_overhead, max_batch,
                                                    try_batch)
from paper_2505_05856_b200.runtime.model import PRESETS

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gpt2-xl")
ap.add_argument("--stages", type=int, default=8)
ap.add_argument("--cap-gib", type=float, default=40.0)
ap.add_argument("--bandwidth-gbs", type=float, default=48.0, help="host link for swaps (GB/s)")
ap.add_argument("--b-max", type=int, default=64)
ap.add_argument("--b-start", type=int, default=1, help="a micro-batch known to fit (resume)")
ap.add_argument("--out", default=None)
ap.add_argument("--host-cap-gib", type=float, default=64.0)
ap.add_argument("--calibrate", action="store_true")
ap.add_argument("--no-gpu", action="store_true")
ap.add_argument("--no-timing", action="store_true")
ap.add_argument("--strategies", default="even_compute,even_compute_memopt,dawnpiper")
ap.add_argument("--time-at", default="", help="STRAT:B[,STRAT:B]: only time those max batches "
                "(margins 0 / 0.1 / 0.2 as the search)")
args = ap.parse_args()
cfg = PRESETS[args.model]
cap = int(args.cap_gib * (1 << 30))
bw = int(args.bandwidth_gbs * 1e9)
host_cap = int(args.host_cap_gib * (1 << 30))
res = {"host_cap_bytes": host_cap, "model": args.model, "stages": args.stages, "cap_bytes": cap,
       "swap_bandwidth_Bps": bw}
overhead = DEFAULT_OVERHEAD
if args.calibrate and not args.no_gpu:
    t0 = time.time()
    overhead, pts = calibrate_overhead(cfg, args.stages)
    res["overhead_calibration"] = {"points": pts, "seconds": round(time.time() - t0, 1)}
    print(json.dumps({"overhead": overhead.to_doc()}), flush=True)
res["overhead"] = overhead.to_doc()
if args.time_at:
    for item in args.time_at.split(","):
        strat, b = item.split(":")
        for margin in (0.0, 0.1, 0.2):
            timed = try_batch(cfg, int(b), args.stages, cap, bw, strat, host_cap=host_cap,
                              margin=margin, overhead=overhead, timing=True)
            if timed.get("feasible"):
                break
        res[strat] = {"max_micro_batch": int(b), "at_max": timed}
        print(json.dumps({"strategy": strat, "at_max": {k: timed.get(k) for k in (
            "b", "margin", "feasible", "samples_per_s_l_gpus", "samples_per_s_l_gpus_model",
            "bottleneck_us", "stage_peak_gib", "reason")}}), flush=True)
    if args.out:
        open(args.out, "w").write(json.dumps(res, indent=1))
    sys.exit(0)
for strat in args.strategies.split(","):
    t0 = time.time()
    best, hist = max_batch(cfg, args.stages, cap, bw, strat, b_max=args.b_max,
                           log=lambda r: print(json.dumps(r), flush=True), host_cap=host_cap,
                           run_gpu=not args.no_gpu, overhead=overhead, b_start=args.b_start)
    res[strat] = {"max_micro_batch": best, "search_s": round(time.time() - t0, 1), "trials": hist}
    if best and not args.no_gpu and not args.no_timing:
        ok = [r for r in hist if r["b"] == best and r.get("feasible")][0]
        timed = try_batch(cfg, best, args.stages, cap, bw, strat, host_cap=host_cap,
                          margin=ok.get("margin", 0.0), overhead=overhead, timing=True)
        res[strat]["at_max"] = timed
        print(json.dumps({"strategy": strat, "at_max": {k: timed.get(k) for k in (
            "b", "feasible", "samples_per_s_l_gpus", "samples_per_s_l_gpus_model", "bottleneck_us",
            "stage_peak_gib", "reason")}}), flush=True)
even = res.get("even_compute", {}).get("max_micro_batch")
dawn = res.get("dawnpiper", {}).get("max_micro_batch")
res["ratio"] = dawn / even if even and dawn is not None else None
summary = {k: v for k, v in res.items() if not isinstance(v, dict) or k == "overhead"}
for strat in args.strategies.split(","):
    summary[f"{strat}_max_b"] = res[strat]["max_micro_batch"]
    summary[f"{strat}_samples_per_s"] = res[strat].get("at_max", {}).get("samples_per_s_l_gpus")
print(json.dumps(summary), flush=True)
if args.out:
    open(args.out, "w").write(json.dumps(res, indent=1))
