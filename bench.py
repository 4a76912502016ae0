#!/usr/bin/env python
"""Throughput of the DawnPiper pipeline-training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): BERT-large (24 x 1024, 16 heads, FFN 4096,
vocab 30522), seq 512, partitioned by this package's planner into an 8-stage
async-1F1B DawnPiper plan, micro-batch b=64, m=32 micro-batches per step
(m = 4l, cli.py:226-228), bf16 compute with fp32 master weights, PipeDream
weight stashing and a per-micro-batch AdamW update.  BASELINE.json leaves b
open ("b swept"); swept sizes 8 / 16 / 32 / 48 / 64 / 74 gave
533 / 612 / 705 / 725 / 734 / 605 samples/s (profiles/r01_bench_*,
profiles/r02_bench_*, profiles/r02_s3/) -- larger micro-batches fill the
tensor cores better (b=64: 128 x 4 pair tiles for the N=1024 GEMMs, 6.9 full
waves on 74 CTA pairs vs 5.2 at b=48) and amortise the per-micro-batch
optimizer step; b=74 runs out of headroom for the allocator.  At N=1 all 8 stages are
co-located on one GPU; at N>1 (torchrun) the plan has l=N stages, one per GPU.

A step = one pipeline iteration (m micro-batches, b*m samples, every forward,
backward and optimizer update).  value = samples / device time of K steps
(CUDA events, max over ranks).  Inputs (weights 1.4 GB + activations) exceed
the 126 MB L2, so no L2 flush is needed between steps.

The JSON line also carries: e2e (same metric through Pipeline.step with token
ids / labels copied H2D from pinned host memory and the loss vector read back
every step), roofline of the dominant kernel (the tcgen05 GEMM: algorithmic
FLOPs / CUDA-event time of every GEMM launch of one instrumented step),
cpu_baseline (the oracle CPU port, bounded sample), clocks sampled during the
timed region, and gpu_launches per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples/sec at 1/2/4/8 stages; max trainable batch under per-GPU mem cap"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="bert-large")
    ap.add_argument("--micro-batch", type=int, default=64)
    ap.add_argument("--stages", type=int, default=0, help="default: 8 at N=1, N otherwise; "
                    "l < N at N>1 runs N/l data-parallel replicas of an l-stage pipeline")
    ap.add_argument("--micro-batches", type=int, default=32)
    ap.add_argument("--capacity-gib", type=float, default=160.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=10)
    ap.add_argument("--cuda-graph", action="store_true",
                    help="replay each iteration as one captured CUDA graph (RunConfig.cuda_graph)")
    ap.add_argument("--memopt-stage", action="store_true",
                    help="instead of the throughput line: run the heaviest-memopt stage of a "
                         "DawnPiper plan under --cap-gib on the GPU and report model vs measured")
    ap.add_argument("--cap-gib", type=float, default=40.0)
    ap.add_argument("--swap-gbs", type=float, default=48.0, help="host link the planner assumes")
    ap.add_argument("--link-aware", action="store_true",
                    help="--memopt-stage: plan with the link-aware eviction costs (beyond the reference)")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks ----

class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons)}
        # "under load": samples drawing more than half the peak power seen
        pmax = max(power) if power else 0
        loaded = sorted(s for s, p in zip(sm, power) if p >= 0.5 * pmax) or sorted(sm)
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": pmax}


# ---------------------------------------------------------------- oracle ----

CPU_SAMPLE = {"micro_batch": 2, "micro_batches": 2}


def committed_profile(model: str, b: int):
    """A B200-measured profile committed under tests/golden/profiles (the
    inputs of the reference-generated large goldens), or None."""
    import gzip
    from paper_2505_05856_b200 import planner as P
    d = ROOT / "tests" / "golden" / "profiles"
    f = d / f"{model}_b{b}.json.gz"
    if not f.exists():
        return None
    return P.graph_from_doc(json.loads(gzip.decompress(f.read_bytes())))


def committed_cuts_profile(model: str, b: int):
    """The committed measured profile of `model` at the micro-batch closest to
    b (relative node times barely move with b), or None: what the reference
    arm plans its stage cuts on."""
    d = ROOT / "tests" / "golden" / "profiles"
    sizes = sorted(int(f.name.split("_b")[1].split(".")[0]) for f in d.glob(f"{model}_b*.json.gz"))
    if not sizes:
        return None, None
    bb = min(sizes, key=lambda x: (abs(x - b), x))
    return committed_profile(model, bb), bb


class CpuPort:
    """The oracle CPU port (fp32 torch, all host threads) of the training step
    on a bounded sample of the workload: the same model and the same stage
    cuts, m micro-batches of b samples in 1F1B order, forward + backward +
    PipeDream AdamW after every backward.  Model construction, parameter init
    and Adam state are built here, outside any timed region; `step()` times
    one training iteration alone."""

    def __init__(self, model_name: str, cuts, b: int = CPU_SAMPLE["micro_batch"],
                 m: int = CPU_SAMPLE["micro_batches"]):
        import torch
        from oracle.train_ref import RefPipeline, dims_from
        from paper_2505_05856_b200.runtime.model import PRESETS, build_nodes, init_params, synthetic_batch
        torch.set_num_threads(os.cpu_count() or 1)
        self.cores = torch.get_num_threads()
        cfg = PRESETS[model_name]
        nodes = build_nodes(cfg)
        ids = [n.id for n in nodes]
        edges = [-1, *cuts, len(ids) - 1]
        stage_nodes = [ids[edges[i] + 1:edges[i + 1] + 1] for i in range(len(edges) - 1)]
        self.ids, self.labels = synthetic_batch(cfg, m, b, seed=0)
        self.ref = RefPipeline(dims_from(cfg, nodes), init_params(cfg, 0), stage_nodes,
                               dict(lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01))
        self.samples = b * m
        self.sample = (f"{m} micro-batches x b={b} of {model_name} s{cfg.seq} through the same "
                       f"{len(stage_nodes)}-stage cuts in 1F1B order: fwd + bwd + AdamW per "
                       f"micro-batch, fp32 torch on CPU (setup excluded)")

    def step(self) -> float:
        t0 = time.perf_counter()
        self.ref.train(self.ids, self.labels)
        return time.perf_counter() - t0


# ---------------------------------------------------------------- ours ------

def gemm_traffic():
    """DRAM bytes (read + write) per GEMM launch from the committed ncu launch list
    of the bench step (profiles/, cold-cache replay), else None."""
    import gzip
    import csv as _csv
    for name in ("r02s3final_launches_step_b64.csv.gz", "r02s3_launches_step_b64.csv.gz",
                 "r02_launches_step.csv.gz", "r01_launches_step_b32.csv.gz"):
        p = ROOT / "profiles" / name
        if p.exists():
            break
    else:
        return None
    try:
        rows = list(_csv.reader(gzip.open(p, "rt")))
        hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
        h = rows[hi]
        ki, ni, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot, ids = 0.0, set()
        for r in rows[hi + 1:]:
            if len(r) > vi and "gemm_kernel" in r[ki] and r[ni].startswith("dram__bytes"):
                tot += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
                ids.add(r[0])
        return {"bytes_per_launch": round(tot / len(ids)), "launches": len(ids),
                "source": f"profiles/{p.name} (ncu dram__bytes_read+write, cold cache)"} if ids else None
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2505_05856_b200 import kernels as K
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
    from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        from paper_2505_05856_b200.runtime.distributed import run_bench_distributed
        return run_bench_distributed(args)

    cfg = PRESETS[args.model]
    b, m = args.micro_batch, args.micro_batches
    stages = args.stages or 8
    # the planner is fed measured B200 per-node times (runtime/profiler.py)
    from paper_2505_05856_b200.runtime.profiler import profile as b200_profile
    t_prof = time.perf_counter()
    g = b200_profile(cfg, b, iters=args.profile_iters, warmup=3)
    t_prof = time.perf_counter() - t_prof
    cap = int(args.capacity_gib * (1 << 30))
    t_plan = time.perf_counter()
    plan = P.plan(g, P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=cap,
                                  bandwidth=64 << 30))
    t_plan = time.perf_counter() - t_plan
    pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False,
                                            cuda_graph=args.cuda_graph))
    ids, labels = synthetic_batch(cfg, m, b, seed=0)
    ids_d, lab_d = ids.cuda(), labels.cuda()
    st = pipe.streams[pipe.stage_dev[0]]
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        pipe.step(ids_d, lab_d)
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs resident in HBM ----
    clocks = Clocks(pipe.stage_dev[0])
    clocks.start()
    l0 = K.INSTR.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        losses = pipe.step(ids_d, lab_d)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    launches = (K.INSTR.launches - l0) // args.steps
    if args.cuda_graph:  # one graph launch per step; the kernels it replays
        launches = pipe.graph_launches
    samples = args.steps * m * b
    value = samples / (ms / 1e3)

    # ---- e2e: host-pinned inputs copied in, loss read back, every step ----
    ids_h, lab_h = ids.pin_memory(), labels.pin_memory()
    loss_h = torch.empty(m, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(st):
            ids_d.copy_(ids_h, non_blocking=True)
            lab_d.copy_(lab_h, non_blocking=True)
        lv = pipe.step(ids_d, lab_d)
        with torch.cuda.stream(st):
            loss_h.copy_(lv, non_blocking=True)
        st.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e = {"value": samples / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": ids.numel() * ids.element_size() + labels.numel() * labels.element_size(),
           "d2h_bytes_per_step": m * 4}

    # ---- roofline of the dominant kernel: every GEMM of one step, event-timed ----
    # (stages chained op by op for this step, so each GEMM is timed without
    # other stages' kernels sharing the SMs)
    K.INSTR.gemm_events = []
    pipe.serialize = True
    pipe.step(ids_d, lab_d)
    torch.cuda.synchronize()
    pipe.serialize = False
    evs = K.INSTR.gemm_events
    K.INSTR.gemm_events = None
    gemm_flops = sum(e[0] for e in evs)
    gemm_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    achieved = gemm_flops / (gemm_ms / 1e3) / 1e12
    traffic = gemm_traffic()
    # the same step's GEMM kernels timed by CUPTI (kernel start to end; the
    # per-GEMM events above also hold the launch gap that programmatic
    # dependent launch otherwise hides)
    cupti = None
    try:
        from torch.profiler import ProfilerActivity, profile
        pipe.serialize = True
        f0 = K.INSTR.gemm_flops
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            pipe.step(ids_d, lab_d)
            torch.cuda.synchronize()
        pipe.serialize = False
        fl = K.INSTR.gemm_flops - f0
        us = sum(e.device_time_total for e in prof.events()
                 if e.device_type.name == "CUDA" and "gemm_kernel" in e.name)
        if us > 0:
            cupti = {"achieved": round(fl / (us / 1e6) / 1e12, 1), "gemm_ms_per_step": round(us / 1e3, 3),
                     "frac": round(fl / (us / 1e6) / 1e12 / peak, 4)}
    except Exception as e:  # the profiler is optional evidence
        cupti = {"error": str(e)[:200]}
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": (traffic or {}).get("bytes_per_launch"),
                "traffic_unit": "bytes per GEMM launch (DRAM read + write)",
                "traffic_source": (traffic or {}).get("source"),
                "kernel": "dpn gemm_kernel (tcgen05, all launches of one step)",
                "launches_per_step": len(evs), "gemm_ms_per_step": round(gemm_ms, 3),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback",
                "cupti_kernel_time": cupti}

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{args.model} s{cfg.seq}, {stages}-stage DawnPiper 1F1B plan "
                               f"co-located on 1 GPU, b={b}, m={m}, weight stashing + AdamW",
                   "model": args.model, "global_batch": b * m, "seq_len": cfg.seq,
                   "micro_batch": b, "micro_batches": m, "stages": stages,
                   "cuts": list(plan.cuts.positions), "parallelism": f"pp{stages} co-located",
                   "profile": f"measured B200 node times ({args.profile_iters} iters, {t_prof:.1f} s); "
                              f"plan {t_plan:.2f} s; graph hash {P.canonical_hash(g)}",
                   "l2": "working set > L2 (no flush needed)",
                   "issue": "one CUDA graph per iteration" if args.cuda_graph else "eager (ctypes launches)"},
        "model_tflops": round(value * cfg.flops_per_sample() / 1e12, 1),
        "e2e": e2e, "roofline": roofline, "gpu_launches": launches, "clocks": clk,
        "losses_last_step": [round(x, 4) for x in losses.tolist()[:4]],
    }
    out["model_vs_measured"] = model_vs_measured(pipe, g, plan, ids_d, lab_d, b, m, value)
    out["planner"] = planner_timing(args.model, b, stages, t_plan)
    if not args.no_cpu_baseline:
        port = CpuPort(args.model, plan.cuts.positions)
        port.step()  # first touch of the fp32 buffers
        dt = port.step()
        out["cpu_baseline"] = {"value": round(port.samples / dt, 4), "unit": UNIT, "cores": port.cores,
                               "kind": "port", "sample": port.sample + f", {dt:.1f} s"}
    print(json.dumps(out), flush=True)


def model_vs_measured(pipe, g, plan, ids_d, lab_d, b: int, m: int, measured: float) -> dict:
    """The cost model (profile + plan + simulate, simulate.py:130-166,
    326-336) beside what the run measures.

    * per stage: forward / backward time of one micro-batch as the planner
      models it (segment times of the measured profile; memopt added_time
      charged to the backward, simulate.py:136-138) vs the stage's mean
      forward / backward in a step with the stages chained op by op (no
      co-located overlap);
    * simulate()'s iteration time and samples/s for the plan on l GPUs (what
      the plan predicts for the 8-GPU deployment);
    * the 1-GPU co-located prediction -- all stages' work on one device:
      b / sum_x (T_x + added_x) -- vs the measured samples/s and the measured
      steady-state iteration time (async_iteration on a traced step)."""
    import torch
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.planner import stage_bounds
    bounds = stage_bounds(plan.cuts, len(g))
    ev: list = []
    pipe.serialize = True
    pipe.step(ids_d, lab_d, ev)
    torch.cuda.synchronize()
    pipe.serialize = False
    per = {}
    for x, j, kind, e0, e1 in ev:
        per.setdefault((x, kind), []).append(e0.elapsed_time(e1) * 1e3)
    stages = []
    for x, (lo, hi) in enumerate(bounds, start=1):
        mf = sum(per[(x, "fwd")]) / len(per[(x, "fwd")])
        mb = sum(per[(x, "bwd")]) / len(per[(x, "bwd")])
        stages.append({"stage": x, "fwd_us_model": g.segment_fwd_time(lo, hi), "fwd_us_measured": round(mf, 1),
                       "bwd_us_model": g.segment_bwd_time(lo, hi) + plan.memopt[x - 1].added_time,
                       "bwd_us_measured": round(mb, 1)})
    # measured steady-state iteration of the real (concurrent) schedule
    ev = []
    t0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(pipe.streams[pipe.stage_dev[0]])
    losses = pipe.step(ids_d, lab_d, ev)
    rep = pipe.report(ev, t0, losses, 0.0)
    sim = P.simulate(plan, g, P.SimConfig(micro_batches=m, schedule=plan.schedule,
                                          bandwidth=plan.config.bandwidth, capacity=plan.config.capacity))
    serial_us = sum(s.time + mo.added_time for s, mo in zip(plan.stages, plan.memopt))
    return {
        "per_stage": stages,
        "simulate_l_gpus": {"stages": len(bounds), "iteration_time_us": round(sim.iteration_time, 1),
                            "samples_per_s": round(b * 1e6 / sim.iteration_time, 1),
                            "bubble_ratio": round(sim.bubble_ratio, 4)},
        "one_gpu": {"model_samples_per_s": round(b * 1e6 / serial_us, 1),
                    "measured_samples_per_s": round(measured, 1),
                    "model_iteration_us": serial_us,
                    "measured_iteration_us": round(rep.iteration_time, 1)},
    }


def planner_timing(model: str, b: int, stages: int, t_live: float) -> dict:
    """Planner wall time: the live plan of this run, and this package's planner
    vs the unmodified reference (dawnplan.plan_with_trace, timed in the dev
    container by oracle/gen_golden_large.py) on the same committed B200
    profile and configuration, with byte-identical plan_json."""
    import gzip
    import hashlib
    from paper_2505_05856_b200 import planner as P
    out = {"live_plan_s": round(t_live, 3)}
    gold = ROOT / "tests" / "golden" / "planner_golden_large.json.gz"
    if not gold.exists():
        return out
    cases = json.loads(gzip.decompress(gold.read_bytes()))["cases"]
    rows = []
    for rec in cases:
        if "plan_json_sha256" not in rec:
            continue
        prof, bsz = rec["profile"].rsplit("_b", 1)
        g = committed_profile(prof, int(bsz))
        cfg = P.PlanConfig(stages=rec["stages"], schedule=rec["schedule"], capacity=rec["capacity"],
                           bandwidth=rec["bandwidth"])
        t0 = time.perf_counter()
        p = P.plan(g, cfg)
        dt = time.perf_counter() - t0
        rows.append({"profile": rec["profile"], "stages": rec["stages"], "capacity": rec["capacity"],
                     "memopt_actions": sum(len(s["memopt"]) for s in rec["plan_doc"]["stages"]),
                     "ours_s": round(dt, 3), "reference_s": rec["reference_plan_s"],
                     "identical": hashlib.sha256(P.plan_json(p).encode()).hexdigest() == rec["plan_json_sha256"]})
    out["vs_reference"] = rows
    out["reference_timing_host"] = "dev container, 8 cores (the reference is not shipped to the GPU box)"
    return out


def run_reference(args):
    """The reference arm: the training step's CPU implementation (the oracle
    port -- the reference `dawnplan` has a planner and an analytic simulator
    but no executor) on all host cores, same model and same DawnPiper stage
    cuts as our arm's workload, each step a bounded sample of it (CPU_SAMPLE).
    The cuts come from planning the committed B200-measured profile of the
    workload with the package planner (byte-identical to the reference's
    plan); setup is outside the timed steps."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    from paper_2505_05856_b200.runtime.model import PRESETS
    cfg = PRESETS[args.model]
    stages = args.stages or (8 if world == 1 else world)
    g, bb = committed_cuts_profile(args.model, args.micro_batch)
    src = f"committed B200-measured profile at b={bb}" if g is not None else "analytic profile"
    if g is None:
        g = profile_graph(cfg, args.micro_batch)
    plan = P.plan(g, P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC,
                                  capacity=int(args.capacity_gib * (1 << 30)), bandwidth=64 << 30))
    port = CpuPort(args.model, plan.cuts.positions)
    for _ in range(args.warmup):
        port.step()
    total = sum(port.step() for _ in range(args.steps))
    value = port.samples * args.steps / total
    out = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": f"{args.model} s{cfg.seq}, {stages}-stage DawnPiper 1F1B plan "
                                  f"(cuts from the {src}), CPU training step "
                                  f"on a bounded sample per step",
                      "model": args.model, "seq_len": cfg.seq, "stages": stages,
                      "cuts": list(plan.cuts.positions), **CPU_SAMPLE},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": port.cores, "kind": "port",
                            "sample": port.sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_memopt_stage(args):
    """The memory plan executing: profile the model on the
    B200 at micro-batch b, plan it for l stages under a per-GPU cap
    (maxbatch.plan_for_cap: the planner gets the cap minus the optimizer state
    its model does not see), then run the stage that evicts the most bytes
    alone on the GPU under the cap with its real 1F1B op list
    (runtime/memprobe.py) and report the planner's charge beside the measured
    backward, swap-in stalls, recompute time, copy GB/s and device peak."""
    from paper_2505_05856_b200.runtime.maxbatch import plan_for_cap
    from paper_2505_05856_b200.runtime.memprobe import heaviest_stage, probe_stage
    from paper_2505_05856_b200.runtime.model import PRESETS
    from paper_2505_05856_b200.runtime.profiler import profile as b200_profile
    cfg = PRESETS[args.model]
    b, stages = args.micro_batch, args.stages or 8
    cap = int(args.cap_gib * (1 << 30))
    g = b200_profile(cfg, b, iters=args.profile_iters, warmup=3)
    t0 = time.perf_counter()
    plan, pcfg = plan_for_cap(cfg, g, stages, cap, int(args.swap_gbs * 1e9), b=b,
                              link_aware=args.link_aware)
    t_plan = time.perf_counter() - t0
    x = heaviest_stage(plan)
    # the executor's memory-faithful defaults, then the throughput knobs
    # Pipeline runs with (RunConfig.d2h_budget / swap_prefetch)
    res = probe_stage(cfg, g, plan, x, b, cap=cap)
    from paper_2505_05856_b200.runtime.pipeline import RunConfig
    rc = RunConfig(micro_batches=1, micro_batch_size=b)
    res_overlap = probe_stage(cfg, g, plan, x, b, cap=cap,
                              swap_knobs={"d2h_budget": rc.d2h_budget, "prefetch_budget": rc.swap_prefetch})
    out = {"mode": "memopt_stage", "model": args.model, "micro_batch": b, "stages": stages,
           "link_aware": args.link_aware,
           "cap_bytes": cap, "planner_capacity": pcfg.capacity, "planner_bandwidth_Bps": pcfg.bandwidth,
           "plan_s": round(t_plan, 3), "cuts": list(plan.cuts.positions),
           "actions_per_stage": [len(m.actions) for m in plan.memopt],
           "host_link_GBps_measured_r01": "57 D2H / 55 H2D (profiles/r01_swap_bw.jsonl)",
           "probe": res, "probe_overlapped": res_overlap}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.memopt_stage:
        return run_memopt_stage(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
