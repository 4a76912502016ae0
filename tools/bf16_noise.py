"""bf16 storage noise floor: gradients of the fp32 oracle vs the same oracle with every node output rounded to bf16.

    python tools/bf16_noise.py tiny-amoeba 4
"""
import sys, torch
sys.path.insert(0, ".")
import oracle.train_ref as T
from paper_2505_05856_b200.runtime.model import PRESETS, build_nodes, init_params, synthetic_batch
name = sys.argv[1]; b = int(sys.argv[2])
cfg = PRESETS[name]; nodes = build_nodes(cfg); init = init_params(cfg, 0)
x, lab = synthetic_batch(cfg, 1, b, seed=3)
def grads(round_bf16):
    ref = T.RefStage(T.dims_from(cfg, nodes), init, [n.id for n in nodes], dict(lr=0.0, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0))
    if round_bf16:
        orig = ref._node
        def rn(nid, env, W, ids, labels):
            y = orig(nid, env, W, ids, labels)
            if nid == "head": return y
            return y + (y.detach().bfloat16().float() - y.detach())   # forward value rounded, gradient straight-through
        ref._node = rn
        # weights rounded too
        ref.params = {k: v.bfloat16().float() for k, v in ref.params.items()}
    ref.forward(1, {}, ids=x[0], labels=lab[0])
    _, env, ver = ref.inflight[1]
    env["head"].backward()
    return {k: v.grad.flatten().clone() for k, v in ver.items()}, float(env["head"])
g32, l32 = grads(False); g16, l16 = grads(True)
print("loss", l32, l16)
cs = sorted((float(torch.dot(g32[k], g16[k]) / (g32[k].norm() * g16[k].norm() + 1e-20)), k) for k in g32)
for c, k in cs[:8]: print(round(c, 4), k)
print("median", cs[len(cs)//2][0])
