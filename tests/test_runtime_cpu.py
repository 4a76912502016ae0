import pathlib
"""Host-side runtime logic that needs no GPU: profile graphs built from the
model definition, the co-located issue order, plan <-> executor tensor naming."""
import json

import pytest

from paper_2505_05856_b200 import planner as P
from paper_2505_05856_b200.runtime.graph import out_tid, profile_graph, stats_tid
from paper_2505_05856_b200.runtime.model import PRESETS, build_nodes, init_params, output_spec
from paper_2505_05856_b200.runtime.pipeline import colocated_order


@pytest.mark.parametrize("name", ["tiny", "tiny-unfused", "bert-base", "bert-large", "gpt2-xl"])
def test_profile_graph_is_a_valid_schema1_profile(name, tmp_path):
    cfg = PRESETS[name]
    g = profile_graph(cfg, 2)
    assert len(g) == 3 + (9 if cfg.fused_attention else 10) * cfg.layers
    f = tmp_path / "p.json"
    P.save_profile(g, f)
    g2 = P.load_profile(f)
    assert P.canonical_hash(g2) == P.canonical_hash(g)
    # canonical order equals the executor's node order
    assert [n.id for n in g.nodes] == [n.id for n in build_nodes(cfg)]
    # every saved tensor names a producer output or LN statistics
    for n in g.nodes:
        for t in n.saved:
            assert t.id in (out_tid(n.id), stats_tid(n.id))


def test_profile_parser_rejects_unknown_fields(tmp_path):
    """The schema rules restated in planner.profile reject unknown node fields."""
    g = profile_graph(PRESETS["tiny"], 2)
    doc = P.profile_doc(g)
    doc["nodes"][0]["extra"] = 1
    with pytest.raises(P.ProfileParseError, match="unknown node field"):
        P.graph_from_doc(doc)


@pytest.mark.skipif(not pathlib.Path("/root/reference/pkg/src").exists(),
                    reason="reference not mounted")
@pytest.mark.parametrize("model,b", [("tiny", 2), ("tiny-t5", 2), ("bert-large", 8),
                                     ("gpt2-xl", 1), ("t5-large", 4), ("amoebanet-d", 16)])
def test_profile_loads_in_the_reference(tmp_path, model, b):
    """Profiles written by the B200 side load in the unmodified reference's
    strict `load_profile` with the same canonical hash."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    import dawnplan
    g = profile_graph(PRESETS[model], b)
    f = tmp_path / "g.json"
    P.save_profile(g, f)
    rg = dawnplan.load_profile(f)
    assert dawnplan.canonical_hash(rg) == P.canonical_hash(g)
    assert len(rg.nodes) == len(g)


def test_param_count_matches_model_definition():
    cfg = PRESETS["bert-large"]
    params = init_params(PRESETS["tiny"], 0)
    assert sum(t.numel() for t in params.values()) == PRESETS["tiny"].n_params()
    assert 330e6 < cfg.n_params() < 370e6
    assert abs(cfg.flops_per_sample() / 1e12 - 1.101) < 0.01


@pytest.mark.parametrize("stages,m", [(1, 1), (2, 3), (4, 16), (8, 32)])
def test_colocated_order_respects_1f1b_and_dependencies(stages, m):
    order = colocated_order(stages, m)
    per_stage = {x: [(k, j) for (s, k, j) in order if s == x] for x in range(1, stages + 1)}
    for x in range(1, stages + 1):
        assert per_stage[x] == [(k, j) for k, j, _ in P.async_ops(stages, m, x)]
    pos = {(s, k, j): i for i, (s, k, j) in enumerate(order)}
    for (s, k, j), i in pos.items():
        if k == "fwd" and s > 1:
            assert pos[(s - 1, "fwd", j)] < i
        if k == "bwd" and s < stages:
            assert pos[(s + 1, "bwd", j)] < i
        if k == "bwd":
            assert pos[(s, "fwd", j)] < i


def test_memopt_actions_name_executor_tensors():
    """Every tensor the planner may evict is one the stage executor can place."""
    cfg = PRESETS["tiny"]
    g = profile_graph(cfg, 2)
    cb = P.compute_balanced(g, 0, len(g) - 1, [1, 1])
    top = max(s.sched_peak for s in P.stage_profiles(g, cb, 2, P.SCHEDULE_ASYNC))
    p = P.plan(g, P.PlanConfig(2, P.SCHEDULE_ASYNC, int(0.55 * top), 50 << 20))
    names = {out_tid(n.id) for n in build_nodes(cfg)} | {stats_tid(n.id) for n in build_nodes(cfg)}
    acts = [a for m in p.memopt for a in m.actions]
    assert acts
    assert all(a.tensor_id in names for a in acts)


@pytest.mark.parametrize("name", ["tiny-t5", "t5-large"])
def test_encdec_profile_graph(name, tmp_path):
    """T5 encoder-decoder: canonical order = executor order; E (enc_ln) feeds
    every cross-attention; the cross-attention's q / kv / P are saved by it."""
    cfg = PRESETS[name]
    g = profile_graph(cfg, 2)
    ids = [n.id for n in g.nodes]
    assert ids == [n.id for n in build_nodes(cfg)]
    assert len(g) == 5 + 9 * cfg.layers + 12 * cfg.dec_layers
    assert ids[:2] == ["embed", "dembed"]
    e = g.nodes[ids.index("enc_ln")]
    assert sorted(e.consumers) == sorted(f"d{i}.xattn" for i in range(cfg.dec_layers))
    x = g.nodes[ids.index("d0.xattn")]
    assert {t.id for t in x.saved} == {"d0.xattn.out", "d0.xattn.q", "d0.xattn.kv", "d0.xattn.lse"}
    P.save_profile(g, tmp_path / "p.json")
    assert P.canonical_hash(P.load_profile(tmp_path / "p.json")) == P.canonical_hash(g)
    params = init_params(cfg, 0) if name == "tiny-t5" else None
    if params is not None:
        assert sum(t.numel() for t in params.values()) == cfg.n_params()
    if name == "t5-large":
        assert abs(cfg.flops_per_sample() / 1e12 - 1.48) < 0.01


@pytest.mark.parametrize("schedule", ["async_1f1b", "sync"])
def test_oracle_encdec_is_partition_invariant(schedule):
    """The CPU oracle's first-iteration first-micro-batch loss does not depend on
    the partition (same weights); the pipelined run must also be finite and
    consistent in shape for a 3-stage T5 split with relayed boundary tensors."""
    import sys
    from pathlib import Path
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.train_ref import reference_train
    from paper_2505_05856_b200.runtime.model import synthetic_batch
    cfg = PRESETS["tiny-t5"]
    nodes = [n.id for n in build_nodes(cfg)]
    ids, labels = synthetic_batch(cfg, 3, 2, seed=0)
    dims = dict(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads, seq=cfg.seq,
                vocab=cfg.vocab, causal=cfg.causal, ln_eps=cfg.ln_eps, dec_layers=cfg.dec_layers,
                tgt_seq=cfg.tgt_seq)
    opt = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    init = init_params(cfg, 0)
    one, _ = reference_train(dims, init, ids, labels, [nodes], opt, schedule=schedule)
    cut = [nodes[:20], nodes[20:33], nodes[33:]]
    three, _ = reference_train(dims, init, ids, labels, cut, opt, schedule=schedule)
    assert abs(one[0][0] - three[0][0]) < 1e-5
    assert abs(one[0][0] - torch.log(torch.tensor(float(cfg.vocab))).item()) < 0.2
    if schedule == "sync":  # one update after all micro-batches: every loss is pre-update
        for a, b in zip(one[0], three[0]):
            assert abs(a - b) < 1e-5


@pytest.mark.parametrize("name", ["tiny-amoeba", "amoebanet-d"])
def test_cnn_profile_graph(name, tmp_path):
    """AmoebaNet-D: valid schema-1 profile in canonical order, cells with skip
    inputs, BN statistics and max-pool argmax saved by their nodes."""
    cfg = PRESETS[name]
    g = profile_graph(cfg, 4)
    assert [n.id for n in g.nodes] == [n.id for n in build_nodes(cfg)]
    P.save_profile(g, tmp_path / "p.json")
    assert P.canonical_hash(P.load_profile(tmp_path / "p.json")) == P.canonical_hash(g)
    kinds = {n.kind for n in build_nodes(cfg)}
    assert {"stem", "bn", "relu", "pw", "dw", "pool", "add", "concat", "gap", "head"} <= kinds
    ids = [n.id for n in g.nodes]
    bn = g.nodes[ids.index("stem.bn")]
    assert "stem.bn.stats" in {t.id for t in bn.saved}
    if name == "amoebanet-d":
        assert 25e6 < cfg.n_params() < 30e6          # ~28M
        assert sum(t.numel() for t in init_params(cfg, 0).values()) == cfg.n_params()


def test_oracle_cnn_is_partition_invariant():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.train_ref import dims_from, reference_train
    from paper_2505_05856_b200.runtime.model import synthetic_batch
    cfg = PRESETS["tiny-amoeba"]
    nodes = build_nodes(cfg)
    ids = [n.id for n in nodes]
    x, labels = synthetic_batch(cfg, 2, 2, seed=0)
    opt = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    d = dims_from(cfg, nodes)
    init = init_params(cfg, 0)
    one, _ = reference_train(d, init, x, labels, [ids], opt)
    k = len(ids) // 3
    three, _ = reference_train(d, init, x, labels, [ids[:k], ids[k:2 * k], ids[2 * k:]], opt)
    assert abs(one[0][0] - three[0][0]) < 1e-4
    import math
    assert abs(one[0][0] - math.log(cfg.classes)) < 1.0


@pytest.mark.parametrize("stages,m", [(1, 1), (2, 3), (4, 8)])
def test_sync_order_is_gpipe(stages, m):
    """The co-located GPipe issue order: per stage exactly sync_ops (all
    forwards, then backwards in reverse micro-batch order), dependencies kept."""
    from paper_2505_05856_b200.runtime.pipeline import sync_order
    order = sync_order(stages, m)
    for x in range(1, stages + 1):
        mine = [(k, j) for (s, k, j) in order if s == x]
        assert mine == [(k, j) for k, j, _ in P.sync_ops(stages, m, x)]
    pos = {(s, k, j): i for i, (s, k, j) in enumerate(order)}
    for (s, k, j), i in pos.items():
        if k == "fwd" and s > 1:
            assert pos[(s - 1, "fwd", j)] < i
        if k == "bwd" and s < stages:
            assert pos[(s + 1, "bwd", j)] < i
