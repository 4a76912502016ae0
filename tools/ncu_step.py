"""One bench-configuration pipeline step inside an NVTX range "timed_step", for
ncu captures filtered with --nvtx --nvtx-include "timed_step/".

    python tools/ncu_step.py [model] [micro_batch] [micro_batches] [serial]
"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
name = sys.argv[1] if len(sys.argv) > 1 else "bert-large"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 32
m = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = PRESETS[name]
g = profile_graph(cfg, b)
plan = P.plan(g, P.PlanConfig(8, P.SCHEDULE_ASYNC, 160 << 30, 64 << 30))
pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, trace=False))
pipe.serialize = len(sys.argv) > 4 and sys.argv[4] == "serial"
ids, lab = synthetic_batch(cfg, m, b)
ids, lab = ids.cuda(), lab.cuda()
pipe.step(ids, lab)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed_step")
pipe.step(ids, lab)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
