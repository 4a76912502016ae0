"""Short BERT-large pipeline run for ncu captures (b=8, 8 stages, m=8, 2 steps)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
name = sys.argv[1] if len(sys.argv) > 1 else "bert-large"
cfg = PRESETS[name]; b, m = 8, 8
g = profile_graph(cfg, b)
plan = P.plan(g, P.PlanConfig(8, P.SCHEDULE_ASYNC, 160 << 30, 64 << 30))
pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False))
ids, lab = synthetic_batch(cfg, m, b); ids, lab = ids.cuda(), lab.cuda()
for _ in range(2):
    pipe.step(ids, lab)
torch.cuda.synchronize()
print("done")
