"""End-to-end 1F1B pipeline on the B200 vs the CPU fp32 oracle.

Same init, same synthetic tokens, same partition and per-stage op order; the
B200 run computes in bf16 (fp32 accumulate / statistics / master weights), so
losses and updated parameters are compared at the north-star bf16 tolerance,
rel 2e-2.  Parameter *updates* (w_final - w_init) are compared by cosine
similarity, which is the sensitive check (weights themselves move by ~lr, and
Adam's normalised steps turn bf16 noise in near-zero gradients into +-lr
element flips, so per-element max-abs is not a meaningful metric here).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

REL = 2e-2
# CNN parameters are compared as one vector: with batch norm over small pixel
# populations and max-pool argmax flips, storing activations in bf16 alone
# moves single-micro-batch gradients of individual parameters to cosine
# 0.82-0.97 (median 0.967) of the fp32 ones -- measured by rounding the fp32
# oracle's node outputs to bf16 (tools/bf16_noise.py); the B200 run shows the
# same spread (tools/debug_cnn_grads.py), and Adam's normalised steps amplify
# it per parameter.  Losses are still compared per micro-batch at REL.
CNN_COS = 0.9


def _setup(name, stages, cap_frac, bandwidth, b=2, m=6, schedule="async_1f1b"):
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    from paper_2505_05856_b200.runtime.model import PRESETS
    cfg = PRESETS[name]
    g = profile_graph(cfg, b)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1] * stages)
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, stages, schedule))
    pc = P.PlanConfig(stages=stages, schedule=schedule, capacity=int(cap_frac * top),
                      bandwidth=bandwidth)
    return cfg, g, P.plan(g, pc)


def _compare(cfg, g, plan, b=2, m=6, steps=2, cos_min=0.95, aggregate=False, seed=3,
             ratio_tol=0.1, lr=1e-3):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.train_ref import reference_train
    from paper_2505_05856_b200.planner import stage_bounds
    from paper_2505_05856_b200.runtime.model import AdamWConfig, build_nodes, init_params, synthetic_batch
    from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig

    opt = AdamWConfig(lr=lr)
    rc = RunConfig(micro_batches=m, micro_batch_size=b, opt=opt, trace=False)
    pipe = Pipeline(cfg, g, plan, rc)
    ids, labels = synthetic_batch(cfg, m, b, seed=seed)
    gpu_losses = []
    for _ in range(steps):
        gpu_losses.append(pipe.step(ids.cuda(), labels.cuda()).tolist())
    torch.cuda.synchronize()

    nodes = [n.id for n in build_nodes(cfg)]
    stage_nodes = [nodes[lo:hi + 1] for lo, hi in stage_bounds(plan.cuts, len(g))]
    from oracle.train_ref import dims_from
    dims = dims_from(cfg, build_nodes(cfg))
    init = init_params(cfg, 0)
    ref_losses, ref_params = reference_train(
        dims, init, ids, labels, stage_nodes,
        dict(lr=opt.lr, beta1=opt.beta1, beta2=opt.beta2, eps=opt.eps, weight_decay=opt.weight_decay),
        steps=steps, schedule=plan.schedule)
    for gl, rl in zip(gpu_losses, ref_losses):
        for a, r in zip(gl, rl):
            assert abs(a - r) <= REL * abs(r), (gl, rl)
    bad = []
    if aggregate:
        # all parameters as one vector (CNN: see CNN_COS)
        got = torch.cat([s.params.master_view(n).float().cpu().flatten()
                         for s in pipe.stages for n in s.params.slots])
        want = torch.cat([ref_params[n].flatten() for s in pipe.stages for n in s.params.slots])
        w0 = torch.cat([init[n].flatten() for s in pipe.stages for n in s.params.slots])
        rel = float((got - want).norm() / want.norm())
        dg, dr = got - w0, want - w0
        cos = float(torch.dot(dg, dr) / (dg.norm() * dr.norm()))
        ratio = float(dg.norm() / dr.norm())
        assert rel <= REL and cos >= cos_min and abs(ratio - 1) <= 0.1, (rel, cos, ratio)
        return gpu_losses
    stats = []
    for s in pipe.stages:
        for name in s.params.slots:
            got = s.params.master_view(name).float().cpu()
            want = ref_params[name]
            w0 = init[name]
            if name.endswith("qkv.bias"):
                # the key bias has an exactly-zero gradient (softmax is invariant to a
                # per-row constant); Adam normalises both sides' rounding noise into
                # +-lr steps of random sign, so only the Q and V biases are comparable
                H = cfg.hidden
                keep = torch.cat([torch.arange(0, H), torch.arange(2 * H, 3 * H)])
                got, want, w0 = got[keep], want[keep], w0[keep]
            elif name.endswith("xattn.kv_bias"):  # same for the cross-attention key bias
                H = cfg.hidden
                got, want, w0 = got[H:], want[H:], w0[H:]
            rel = float((got - want).norm() / (want.norm() + 1e-12))
            dg = (got - w0).flatten()
            dr = (want - w0).flatten()
            cos = float(torch.dot(dg, dr) / (dg.norm() * dr.norm() + 1e-12)) if dr.norm() > 0 else 1.0
            ratio = float(dg.norm() / (dr.norm() + 1e-12))
            # parameters with a non-zero init: relative Frobenius error <= REL.
            # zero-init parameters (biases, LN beta) *are* their update, whose
            # bf16-vs-fp32 Adam noise is a few %: judged with every parameter on
            # the update's direction (cos) and magnitude (norm ratio).
            stats.append((name, round(rel, 5), round(cos, 4), round(ratio, 4)))
            if (w0.norm() > 0 and rel > REL) or cos < cos_min or abs(ratio - 1) > ratio_tol:
                bad.append((name, round(rel, 5), round(cos, 4), round(ratio, 4)))
    worst = sorted(stats, key=lambda r: -r[1])[:3]
    print(f"{cfg.name}: worst rel {worst}; min cos {min(r[2] for r in stats):.4f}")
    assert not bad, bad
    return gpu_losses


@pytest.mark.parametrize("stages", [1, 2, 4])
def test_pipeline_matches_oracle_no_memopt(stages):
    cfg, g, plan = _setup("tiny", stages, 4.0, 16 << 30)
    assert all(not m.actions for m in plan.memopt)
    _compare(cfg, g, plan)


def test_pipeline_matches_oracle_causal_three_stages():
    cfg, g, plan = _setup("tiny-causal", 3, 4.0, 16 << 30)
    _compare(cfg, g, plan)


@pytest.mark.parametrize("stages", [2, 3])
def test_pipeline_unfused_attention_vocabulary(stages):
    """The reference vocabulary's materialised `score` + `attn` pair."""
    cfg, g, plan = _setup("tiny-unfused", stages, 4.0, 16 << 30)
    assert any(n.id.endswith(".score") for n in g.nodes)
    _compare(cfg, g, plan)


def test_pipeline_memopt_causal_four_stages():
    cfg, g, plan = _setup("tiny-causal", 4, 0.5, 16 << 30)
    assert any(m.actions for m in plan.memopt)
    _compare(cfg, g, plan)


@pytest.mark.parametrize("frac,bw", [(0.6, 16 << 30), (0.6, 50 << 20), (0.7, 16 << 30)])
def test_pipeline_executes_memopt_actions(frac, bw):
    """A tight capacity makes the planner pick swaps (fast link) and recomputes
    (slow link); the run must execute them and still match the oracle."""
    cfg, g, plan = _setup("tiny", 2, frac, bw)
    kinds = {a.kind for m in plan.memopt for a in m.actions}
    assert kinds, "expected memopt actions at this capacity"
    _compare(cfg, g, plan)


@pytest.mark.parametrize("name,stages", [("tiny", 1), ("tiny", 2), ("tiny-causal", 3)])
def test_pipeline_sync_gpipe_matches_oracle(name, stages):
    """GPipe (sync) schedule: all forwards, reverse-order backwards, gradients
    accumulated over the m micro-batches and one AdamW step per iteration."""
    cfg, g, plan = _setup(name, stages, 4.0, 16 << 30, schedule="sync")
    assert plan.schedule == "sync"
    _compare(cfg, g, plan)


def test_pipeline_sync_with_memopt():
    cfg, g, plan = _setup("tiny", 2, 0.6, 16 << 30, schedule="sync")
    assert any(m.actions for m in plan.memopt)
    _compare(cfg, g, plan)


@pytest.mark.parametrize("stages", [1, 2, 3, 4])
def test_pipeline_t5_encoder_decoder(stages):
    """T5-style encoder-decoder (BASELINE configs[3] at tiny size): relayed
    boundary tensors (decoder layer-0 sub-block outputs through the encoder
    stages, E through the decoder stages), cross-attention, two sequence lengths."""
    cfg, g, plan = _setup("tiny-t5", stages, 4.0, 16 << 30)
    _compare(cfg, g, plan)


def test_pipeline_t5_memopt_and_sync():
    cfg, g, plan = _setup("tiny-t5", 3, 0.6, 16 << 30)
    assert any(m.actions for m in plan.memopt)
    _compare(cfg, g, plan)
    cfg, g, plan = _setup("tiny-t5", 2, 4.0, 16 << 30, schedule="sync")
    _compare(cfg, g, plan)


@pytest.mark.parametrize("stages", [1, 2, 4])
def test_pipeline_amoebanet(stages):
    """AmoebaNet-D-style CNN (BASELINE configs[4] at tiny size): stem conv, BN,
    depthwise-separable convolutions, pooling, concat cells with skip inputs."""
    cfg, g, plan = _setup("tiny-amoeba", stages, 4.0, 16 << 30, b=4)
    _compare(cfg, g, plan, b=4, m=6, cos_min=CNN_COS, aggregate=True)


def test_pipeline_amoebanet_memopt_and_sync():
    cfg, g, plan = _setup("tiny-amoeba", 3, 0.6, 16 << 30, b=4)
    assert any(m.actions for m in plan.memopt)
    _compare(cfg, g, plan, b=4, m=6, cos_min=CNN_COS, aggregate=True)
    cfg, g, plan = _setup("tiny-amoeba", 2, 4.0, 16 << 30, b=4, schedule="sync")
    _compare(cfg, g, plan, b=4, m=4, cos_min=CNN_COS, aggregate=True)


def test_pipeline_middle_stage_relays_several_tensors():
    """A one-node middle stage (d0.ln1, cuts 2|3) receives embed.out and
    b0.ln1.out, which it only passes on, besides its own input: every relayed
    tensor must survive until the stage's sends (regression: each delivery used
    to drop the previously delivered send-only tensors of the same micro-batch)."""
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200.runtime.graph import profile_graph
    from paper_2505_05856_b200.runtime.model import PRESETS
    cfg = PRESETS["tiny-t5"]
    g = profile_graph(cfg, 2)
    pc = P.PlanConfig(stages=4, schedule="async_1f1b", capacity=1 << 40, bandwidth=16 << 30)
    plan = P.plan_from_cuts(g, pc, (2, 3, 20))
    _compare(cfg, g, plan)
