import sys, collections, torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import planner as P, kernels as K
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
cfg = PRESETS["bert-large"]; b, m = 8, 16
g = profile_graph(cfg, b)
plan = P.plan(g, P.PlanConfig(8, P.SCHEDULE_ASYNC, 160 << 30, 64 << 30))
pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False))
pipe.serialize = True  # per-GEMM times without other stages sharing the SMs
ids, lab = synthetic_batch(cfg, m, b); ids, lab = ids.cuda(), lab.cuda()
for _ in range(2): pipe.step(ids, lab)
K.INSTR.gemm_events = []
pipe.step(ids, lab); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0, 0])
for f, a, c, key in K.INSTR.gemm_events:
    r = agg[key]; r[0] += 1; r[1] += a.elapsed_time(c); r[2] += f
tot = sum(r[1] for r in agg.values())
print(f"total gemm {tot:.1f} ms")
for key, (n, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:8.2f} ms {n:5d}x {ms/n*1e3:8.1f} us {fl/(ms/1e3)/1e12:7.1f} TF/s  M,N,K,Z,amn,bmn,f32={key}")
