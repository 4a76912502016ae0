import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_pipeline_gpu import _setup
from oracle.train_ref import reference_train
from paper_2505_05856_b200.planner import stage_bounds
from paper_2505_05856_b200.runtime.model import AdamWConfig, build_nodes, init_params, synthetic_batch
from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
for stages, m, steps in ((2, 1, 3), (2, 2, 2), (2, 3, 2), (2, 6, 2)):
    cfg, g, plan = _setup("tiny", stages, 4.0, 16 << 30)
    b = 2
    opt = AdamWConfig(lr=1e-3)
    pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=m, micro_batch_size=b, opt=opt, trace=False))
    ids, labels = synthetic_batch(cfg, m, b, seed=3)
    gl = [pipe.step(ids.cuda(), labels.cuda()).tolist() for _ in range(steps)]
    nodes = [n.id for n in build_nodes(cfg)]
    sn = [nodes[lo:hi + 1] for lo, hi in stage_bounds(plan.cuts, len(g))]
    dims = dict(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads, seq=cfg.seq, vocab=cfg.vocab, causal=cfg.causal, ln_eps=cfg.ln_eps)
    rl, rp = reference_train(dims, init_params(cfg, 0), ids, labels, sn, dict(lr=1e-3, beta1=.9, beta2=.999, eps=1e-8, weight_decay=.01), steps=steps)
    print("stages", stages, "m", m, "cuts", plan.cuts.positions)
    for a, r in zip(gl, rl): print("  gpu", [round(x, 4) for x in a], "\n  ref", [round(x, 4) for x in r])
    for s in pipe.stages:
        for name in list(s.params.slots)[:40]:
            got = s.params.master_view(name).float().cpu(); want = rp[name]; i0 = init_params(cfg, 0)[name]
            dg, dr = (got - i0).flatten(), (want - i0).flatten()
            cos = float(torch.dot(dg, dr) / (dg.norm() * dr.norm() + 1e-12))
            if cos < 0.98: print("   ", name, "cos", round(cos, 4), "norms", float(dg.norm()), float(dr.norm()))
