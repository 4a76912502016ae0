"""Per-parameter gradient agreement (one micro-batch) between the B200 executor and the CPU oracle."""
import sys
import torch
sys.path.insert(0, ".")
from oracle.train_ref import RefStage, dims_from
from paper_2505_05856_b200 import _lib
from paper_2505_05856_b200.planner.memplan import MemOptPlan
from paper_2505_05856_b200.runtime.graph import profile_graph
from paper_2505_05856_b200.runtime.model import PRESETS, AdamWConfig, build_nodes, init_params, synthetic_batch
from paper_2505_05856_b200.runtime.stage import StageExecutor
name = sys.argv[1] if len(sys.argv) > 1 else "tiny-amoeba"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = PRESETS[name]
_lib.init_device(0)
nodes = build_nodes(cfg)
g = profile_graph(cfg, b)
init = init_params(cfg, 0)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
ex = StageExecutor(cfg=cfg, g=g, nodes=nodes, lo=0, hi=len(nodes) - 1, stage=1, stages=1, micro_batch=b,
                   memopt=MemOptPlan(), init=init, device=dev, stream=st, opt=AdamWConfig(lr=0.0, weight_decay=0.0))
x, lab = synthetic_batch(cfg, 1, b, seed=3)
loss = torch.zeros(1, device=dev)
with torch.cuda.stream(st):
    ex.forward(1, ids=x[0].cuda(), labels=lab[0].cuda(), loss_out=loss)
    ex.backward(1)
torch.cuda.synchronize()
ref = RefStage(dims_from(cfg, nodes), init, [n.id for n in nodes], dict(lr=0.0, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0))
env = ref.forward(1, {}, ids=x[0], labels=lab[0])
leaves, envd, version = ref.inflight[1]
envd["head"].backward()
print("loss", loss.item(), float(envd["head"]))
rows = []
for pname, s in ex.params.slots.items():
    gg = ex.params.grad[s.offset:s.offset + s.numel].float().cpu()
    gr = version[pname].grad.flatten()
    cos = float(torch.dot(gg, gr) / (gg.norm() * gr.norm() + 1e-20))
    rel = float((gg - gr).norm() / (gr.norm() + 1e-20))
    rows.append((cos, rel, pname, float(gr.norm())))
rows.sort()
for r in rows[:25]:
    print(f"cos {r[0]:.4f} rel {r[1]:.4f} |g| {r[3]:.3e} {r[2]}")
print("median cos", rows[len(rows) // 2][0])
