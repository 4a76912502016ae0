import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_pipeline_gpu import _setup
from oracle.train_ref import reference_train
from paper_2505_05856_b200.planner import stage_bounds
from paper_2505_05856_b200.runtime.model import AdamWConfig, build_nodes, init_params, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
for lr in (0.0, 1e-3):
  for stages in (1, 2, 4):
    m, steps, b = 4, 2, 2
    cfg, g, plan = _setup("tiny", stages, 4.0, 16 << 30)
    opt = AdamWConfig(lr=lr, weight_decay=0.0)
    pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, opt=opt, trace=False))
    torch.cuda.synchronize()
    ids, labels = synthetic_batch(cfg, m, b, seed=3)
    gl = [pipe.step(ids.cuda(), labels.cuda()).tolist() for _ in range(steps)]
    nodes = [n.id for n in build_nodes(cfg)]
    sn = [nodes[lo:hi + 1] for lo, hi in stage_bounds(plan.cuts, len(g))]
    dims = dict(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads, seq=cfg.seq, vocab=cfg.vocab, causal=cfg.causal, ln_eps=cfg.ln_eps)
    rl, rp = reference_train(dims, init_params(cfg, 0), ids, labels, sn, dict(lr=lr, beta1=.9, beta2=.999, eps=1e-8, weight_decay=0.0), steps=steps)
    print("lr", lr, "stages", stages, "cuts", plan.cuts.positions, flush=True)
    for a, r in zip(gl, rl): print("  gpu", [round(x, 4) for x in a], "\n  ref", [round(x, 4) for x in r])
    if lr > 0:
        worst = []
        for s in pipe.stages:
            for name in s.params.slots:
                got = s.params.master_view(name).float().cpu(); want = rp[name]; i0 = init_params(cfg, 0)[name]
                dg, dr = (got - i0).flatten(), (want - i0).flatten()
                worst.append((round(float(torch.dot(dg, dr) / (dg.norm() * dr.norm() + 1e-12)), 3), name))
        print("  worst cos", sorted(worst)[:6])
