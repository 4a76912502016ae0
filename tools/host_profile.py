"""Host issue cost of one pipeline step: wall time to enqueue vs GPU time, + cProfile."""
import sys, time, cProfile, pstats, io, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
name = sys.argv[1] if len(sys.argv) > 1 else "bert-large"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = int(sys.argv[3]) if len(sys.argv) > 3 else 32
stages = int(sys.argv[4]) if len(sys.argv) > 4 else 8
cfg = PRESETS[name]
g = profile_graph(cfg, b)
plan = P.plan(g, P.PlanConfig(stages, P.SCHEDULE_ASYNC, 160 << 30, 64 << 30))
pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False))
ids, lab = synthetic_batch(cfg, m, b); ids, lab = ids.cuda(), lab.cuda()
for _ in range(3): pipe.step(ids, lab)
torch.cuda.synchronize()
st = pipe.streams[0]
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(st); t0 = time.perf_counter(); pipe.step(ids, lab); t1 = time.perf_counter(); e1.record(st)
torch.cuda.synchronize()
print(f"issue {1e3*(t1-t0):.1f} ms, gpu {e0.elapsed_time(e1):.1f} ms")
pr = cProfile.Profile(); pr.enable(); pipe.step(ids, lab); torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
