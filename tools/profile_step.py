"""Kernel-time breakdown of one pipeline step (torch.profiler / CUPTI)."""
import sys, json, collections, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
name = sys.argv[1] if len(sys.argv) > 1 else "bert-large"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = PRESETS[name]; g = profile_graph(cfg, b)
plan = P.plan(g, P.PlanConfig(8, P.SCHEDULE_ASYNC, 160 << 30, 64 << 30))
pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False))
pipe.serialize = len(sys.argv) > 4 and sys.argv[4] == "serial"
ids, lab = synthetic_batch(cfg, m, b); ids, lab = ids.cuda(), lab.cuda()
for _ in range(2): pipe.step(ids, lab)
torch.cuda.synchronize()
st = pipe.streams[0]
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(st); pipe.step(ids, lab); e1.record(st); torch.cuda.synchronize()
print(f"event-timed step (no profiler): {e0.elapsed_time(e1):.1f} ms")
from torch.profiler import profile, ProfilerActivity
import time
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter(); pipe.step(ids, lab); torch.cuda.synchronize(); wall = time.perf_counter() - t0
tot = collections.Counter(); cnt = collections.Counter()
kern = [e for e in prof.events() if e.device_type.name == "CUDA"]
for e in kern:
    key = e.name[:90]
    tot[key] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    cnt[key] += 1
busy = sum(tot.values())
print(f"wall {wall*1e3:.1f} ms, kernel busy {busy/1e3:.1f} ms, kernels {sum(cnt.values())}")
for k, v in tot.most_common(25):
    print(f"{v/1e3:9.2f} ms {cnt[k]:6d}  {v/cnt[k]:8.1f} us  {k}")
