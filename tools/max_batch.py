"""Max trainable micro-batch under a per-GPU cap: DawnPiper plan vs even-compute split.

    python tools/max_batch.py [--model gpt2-xl] [--stages 8] [--cap-gib 40] [--no-gpu]
"""
import argparse, json, sys, time
sys.path.insert(0, ".")
from paper_2505_05856_b200.runtime.maxbatch import max_batch
from paper_2505_05856_b200.runtime.model import PRESETS

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="gpt2-xl")
ap.add_argument("--stages", type=int, default=8)
ap.add_argument("--cap-gib", type=float, default=40.0)
ap.add_argument("--bandwidth-gbs", type=float, default=48.0, help="host link for swaps (GB/s)")
ap.add_argument("--b-max", type=int, default=64)
ap.add_argument("--out", default=None)
ap.add_argument("--host-cap-gib", type=float, default=96.0)
ap.add_argument("--no-gpu", action="store_true")
args = ap.parse_args()
cfg = PRESETS[args.model]
cap = int(args.cap_gib * (1 << 30))
res = {"host_cap_bytes": int(args.host_cap_gib * (1 << 30)), "model": args.model, "stages": args.stages, "cap_bytes": cap, "swap_bandwidth_Bps": int(args.bandwidth_gbs * 1e9)}
for strat in ("even_compute", "even_compute_memopt", "dawnpiper"):
    t0 = time.time()
    best, hist = max_batch(cfg, args.stages, cap, int(args.bandwidth_gbs * 1e9), strat, b_max=args.b_max,
                           log=lambda r: print(json.dumps(r), flush=True),
                           host_cap=int(args.host_cap_gib * (1 << 30)), run_gpu=not args.no_gpu)
    res[strat] = {"max_micro_batch": best, "search_s": round(time.time() - t0, 1), "trials": hist}
res["ratio"] = (res["dawnpiper"]["max_micro_batch"] / res["even_compute"]["max_micro_batch"]
                if res["even_compute"]["max_micro_batch"] else None)
print(json.dumps({k: v for k, v in res.items() if k not in ("even_compute", "dawnpiper")} |
                 {"even_compute_max_b": res["even_compute"]["max_micro_batch"],
                  "even_compute_memopt_max_b": res["even_compute_memopt"]["max_micro_batch"],
                  "dawnpiper_max_b": res["dawnpiper"]["max_micro_batch"]}))
if args.out:
    open(args.out, "w").write(json.dumps(res, indent=1))
