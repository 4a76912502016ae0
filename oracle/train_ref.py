"""CPU fp32 restatement of the pipeline training step -- TEST ORACLE ONLY.

This file is test infrastructure: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg may import it, and only as the
checker or the timed CPU baseline.  It never runs on the product path.

Parity status: UNPINNED.  The reference (dawnplan) has no model, optimizer or
loss code, so there is no reference output to pin these
numerics to; this restatement fixes the semantics instead:

  * model: pre-LN transformer blocks
        h1 = LN1(x); [q|k|v] = h1 Wqkv^T + bqkv; P = softmax(q k^T / sqrt(d) [causal])
        ctx = P v; y = ctx Wo^T + bo + x; h2 = LN2(y); f = h2 W1^T + b1
        g = gelu_tanh(f); z = g W2^T + b2; out = z + y
    embed = tok[ids] + pos[t]; head = LN_f then logits = h Wh[:V]^T,
    loss = mean-over-tokens cross entropy per micro-batch;
  * encoder-decoder (T5-large config): encoder blocks as above (non-causal) ->
    E = enc_ln(x); decoder input dembed(tgt ids); decoder block = causal
    self-attention sub-block, then c = lnx(y); q = c Wq^T + bq;
    kv = E Wkv^T + bkv; ctx = softmax(q k^T / sqrt(d)) v; y2 = ctx Wo^T + bo + y;
    then the FFN sub-block; lnf / head over the target tokens.  ids per
    micro-batch are the b*s source ids followed by the b*t target ids;
  * CNN (AmoebaNet-D config): the node structure (kind, inputs, geometry) is
    given as data in dims["graph"]; each kind's math is restated here with
    torch.nn.functional on NCHW fp32 tensors -- stem 3x3 convolution,
    training-mode batch norm (biased variance), ReLU, 1x1 convolution,
    depthwise 3x3 convolution, 3x3 max / average pooling (average excludes
    padding), add, channel concat, global average pool, FC + cross entropy;
  * schedule: per stage x of l, the 1F1B op list of simulate.py:211-222
    (restated below as `one_f_one_b`);
  * weight stashing (PipeDream): a forward uses the stage's newest weights and
    its backward differentiates through that same version; every backward is
    followed by an AdamW step on the fp32 master weights;
  * sync schedule (GPipe, simulate.py:169-208): all forwards, then backwards in
    reverse micro-batch order with one weight version; gradients accumulate
    and one AdamW step on their mean ends the iteration;
  * AdamW: torch.optim.AdamW semantics (decoupled weight decay, bias
    correction), applied to every parameter.

Everything is computed in fp32 with torch autograd on the host CPU.
"""

from __future__ import annotations

import math
from typing import Dict, List, Sequence, Tuple

import torch
import torch.nn.functional as F


def one_f_one_b(stages: int, m: int, x: int) -> List[Tuple[str, int]]:
    """simulate.py:211-222: min(l-x, m) warm-up forwards, (F, B) pairs, drain."""
    warm = min(stages - x, m)
    ops = [("fwd", j) for j in range(1, warm + 1)]
    k = 0
    while warm + k < m:
        k += 1
        ops.append(("fwd", warm + k))
        ops.append(("bwd", k))
    ops += [("bwd", j) for j in range(k + 1, m + 1)]
    return ops


def node_ids(layers: int, fused: bool = True) -> List[str]:
    """Node ids; with fused attention `attn` reads qkv directly (no `score`)."""
    ids = ["embed"]
    block = ("ln1", "qkv", "attn", "proj", "ln2", "fc1", "gelu", "fc2", "add") if fused else \
        ("ln1", "qkv", "score", "attn", "proj", "ln2", "fc1", "gelu", "fc2", "add")
    for b in range(layers):
        ids += [f"b{b}.{k}" for k in block]
    return ids + ["lnf", "head"]


def _inputs(nid: str, d: dict) -> Tuple[str, ...]:
    if "graph" in d:
        return tuple(d["graph"][nid][1])
    layers, dec = d["layers"], d.get("dec_layers", 0)
    fused = d.get("fused_attention", True)
    if nid in ("embed", "dembed"):
        return ()
    if nid == "enc_ln":
        return (f"b{layers - 1}.add",)
    if nid == "lnf":
        return (f"d{dec - 1}.add",) if dec else (f"b{layers - 1}.add",)
    if nid == "head":
        return ("lnf",)
    b, k = nid.split(".")
    blk = int(b[1:])
    if b[0] == "d":
        x = "dembed" if blk == 0 else f"d{blk - 1}.add"
    else:
        x = "embed" if blk == 0 else f"b{blk - 1}.add"
    p = f"{b[0]}{blk}."
    y = p + "xproj" if b[0] == "d" else p + "proj"
    return {
        "ln1": (x,), "qkv": (p + "ln1",), "score": (p + "qkv",),
        "attn": (p + "qkv",) if fused else (p + "score", p + "qkv"),
        "proj": (p + "attn", x), "lnx": (p + "proj",), "xattn": (p + "lnx", "enc_ln"),
        "xproj": (p + "xattn", p + "proj"), "ln2": (y,), "fc1": (p + "ln2",),
        "gelu": (p + "fc1",), "fc2": (p + "gelu",), "add": (p + "fc2", y),
    }[k]


def _mha(q, k, v, b: int, A: int, causal: bool) -> torch.Tensor:
    """Multi-head attention over [b*t, H] q and [b*s, H] k, v -> [b*t, H]."""
    H = q.shape[1]
    hd = H // A
    t, s = q.shape[0] // b, k.shape[0] // b
    qh = q.reshape(b, t, A, hd).transpose(1, 2)
    kh = k.reshape(b, s, A, hd).transpose(1, 2)
    vh = v.reshape(b, s, A, hd).transpose(1, 2)
    sc = (qh @ kh.transpose(-1, -2)) / math.sqrt(hd)
    if causal:
        sc = sc.masked_fill(torch.ones(t, s, dtype=torch.bool).triu(1), float("-inf"))
    return (torch.softmax(sc, -1) @ vh).transpose(1, 2).reshape(b * t, H)


class RefStage:
    def __init__(self, dims: dict, init: Dict[str, torch.Tensor], nodes: Sequence[str], opt: dict,
                 sync_m: int = 0):
        self.d = dims
        self.nodes = list(nodes)
        self.params = {k: v.detach().clone().float() for k, v in init.items()
                       if k.rsplit(".", 1)[0] in self.nodes}
        self.exp_avg = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.exp_sq = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.step = 0
        self.opt = opt
        self.inflight: Dict[int, tuple] = {}
        self.sync_m = sync_m  # > 0: GPipe, accumulate over sync_m micro-batches
        self.gacc = {k: torch.zeros_like(v) for k, v in self.params.items()}

    def _cnn_node(self, nid: str, env, W, images, labels) -> torch.Tensor:
        d = self.d
        kind, inputs, a = d["graph"][nid]
        ins = [env[u] for u in inputs]
        w = lambda pn: W[f"{nid}.{pn}"]
        b = labels.numel()

        def nchw(t, H, Wd):
            return t.reshape(b, H, Wd, -1).permute(0, 3, 1, 2)

        def flat(t):
            return t.permute(0, 2, 3, 1).reshape(-1, t.shape[1])

        if kind == "stem":
            x = nchw(images.float(), a["H"], a["W"])
            wt = w("weight").reshape(a["C"], 3, 3, a["Cin"]).permute(0, 3, 1, 2)
            return flat(F.conv2d(x, wt, stride=a["stride"], padding=1))
        if kind == "bn":
            return F.batch_norm(ins[0], None, None, w("gamma"), w("beta"), training=True,
                                eps=d["ln_eps"])
        if kind == "relu":
            return torch.relu(ins[0])
        if kind == "pw":
            return ins[0] @ w("weight").t()
        if kind == "dw":
            x = nchw(ins[0], a["H"], a["W"])
            return flat(F.conv2d(x, w("weight").reshape(a["C"], 1, 3, 3), stride=a["stride"],
                                 padding=1, groups=a["C"]))
        if kind == "pool":
            x = nchw(ins[0], a["H"], a["W"])
            if a["mode"] == 0:
                return flat(F.max_pool2d(x, 3, a["stride"], 1))
            return flat(F.avg_pool2d(x, 3, a["stride"], 1, count_include_pad=False))
        if kind == "add":
            return ins[0] + ins[1]
        if kind == "concat":
            return torch.cat(ins, 1)
        if kind == "gap":
            return ins[0].reshape(b, a["H"] * a["W"], -1).mean(1)
        if kind == "head":
            logits = ins[0] @ w("weight")[:d["vocab"]].t()
            return F.cross_entropy(logits, labels.long())
        raise ValueError(kind)

    def _node(self, nid: str, env: Dict[str, torch.Tensor], W: Dict[str, torch.Tensor],
              ids, labels) -> torch.Tensor:
        d = self.d
        if "graph" in d:
            return self._cnn_node(nid, env, W, ids, labels)
        H, A, s = d["hidden"], d["heads"], d["seq"]
        hd = H // A
        kind = nid.split(".")[-1] if "." in nid else nid
        fused = d.get("fused_attention", True)
        ins = [env[u] for u in _inputs(nid, d)]
        w = lambda pn: W[f"{nid}.{pn}"]
        dec = nid.startswith("d") and nid != "dembed"  # decoder block node
        T = d.get("tgt_seq", 0)
        if T and (dec or nid in ("dembed",)):
            s = T
        causal = True if dec else (d["causal"] and not T)
        b = ids.numel() // (d["seq"] + T)
        if kind in ("embed", "dembed"):
            src = ids[:b * d["seq"]] if kind == "embed" else ids[b * d["seq"]:]
            M = src.numel()
            return w("tok")[src.long()] + w("pos")[torch.arange(M) % s]
        if kind in ("ln1", "ln2", "lnf", "enc_ln", "lnx"):
            return F.layer_norm(ins[0], (H,), w("gamma"), w("beta"), d["ln_eps"])
        if kind in ("qkv", "fc1", "fc2"):
            return ins[0] @ w("weight").t() + w("bias")
        if kind in ("proj", "xproj"):
            return ins[0] @ w("weight").t() + w("bias") + ins[1]
        if kind == "xattn":
            q = ins[0] @ w("q_weight").t() + w("q_bias")
            kv = ins[1] @ w("kv_weight").t() + w("kv_bias")
            return _mha(q, kv[:, :H], kv[:, H:], b, A, False)
        if kind == "gelu":
            return F.gelu(ins[0], approximate="tanh")
        if kind == "add":
            return ins[0] + ins[1]
        if kind == "score":
            qkv = ins[0]
            b = qkv.shape[0] // s
            q = qkv[:, :H].reshape(b, s, A, hd).transpose(1, 2)
            k = qkv[:, H:2 * H].reshape(b, s, A, hd).transpose(1, 2)
            sc = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
            if causal:
                sc = sc.masked_fill(torch.ones(s, s, dtype=torch.bool).triu(1), float("-inf"))
            return torch.softmax(sc, -1)
        if kind == "attn" and fused:
            qkv = ins[0]
            return _mha(qkv[:, :H], qkv[:, H:2 * H], qkv[:, 2 * H:], b, A, causal)
        if kind == "attn":
            P, qkv = ins
            b = qkv.shape[0] // s
            v = qkv[:, 2 * H:].reshape(b, s, A, hd).transpose(1, 2)
            return (P @ v).transpose(1, 2).reshape(b * s, H)
        if kind == "head":
            logits = ins[0] @ w("weight")[:d["vocab"]].t()
            return F.cross_entropy(logits, labels.long())
        raise ValueError(nid)

    def forward(self, j: int, recv: Dict[str, torch.Tensor], ids=None, labels=None):
        version = {k: v.detach().clone().requires_grad_(True) for k, v in self.params.items()}
        env = {k: t.detach().clone().requires_grad_(True) for k, t in recv.items()}
        leaves = dict(env)
        for nid in self.nodes:
            env[nid] = self._node(nid, env, version, ids, labels)
        self.inflight[j] = (leaves, env, version)
        return env

    def backward(self, j: int, out_grads: Dict[str, torch.Tensor], send_ids: Sequence[str]):
        leaves, env, version = self.inflight.pop(j)
        roots, grads = [], []
        if "head" in env:
            roots.append(env["head"])
            grads.append(torch.ones(()))
        for k, gk in out_grads.items():
            roots.append(env[k])
            grads.append(gk)
        torch.autograd.backward(roots, grads)
        g = {k: (v.grad if v.grad is not None else torch.zeros_like(v)) for k, v in version.items()}
        if self.sync_m:
            for k, gk in g.items():
                self.gacc[k] += gk
        else:
            self._adamw(g)
        return {k: leaves[k].grad.detach() for k in leaves if leaves[k].grad is not None}

    def flush(self) -> None:
        """GPipe: one AdamW step on the mean of the accumulated gradients."""
        if self.sync_m:
            self._adamw({k: v / self.sync_m for k, v in self.gacc.items()})
            for v in self.gacc.values():
                v.zero_()

    def _adamw(self, g: Dict[str, torch.Tensor]) -> None:
        o = self.opt
        self.step += 1
        b1, b2 = o["beta1"], o["beta2"]
        bc1, bc2 = 1 - b1 ** self.step, 1 - b2 ** self.step
        for k, p in self.params.items():
            gk = g[k]
            self.exp_avg[k].mul_(b1).add_(gk, alpha=1 - b1)
            self.exp_sq[k].mul_(b2).addcmul_(gk, gk, value=1 - b2)
            p.mul_(1 - o["lr"] * o["weight_decay"])
            denom = (self.exp_sq[k] / bc2).sqrt().add_(o["eps"])
            p.addcdiv_(self.exp_avg[k] / bc1, denom, value=-o["lr"])


def boundary(stage_nodes: List[List[str]], x: int, dims: dict) -> List[str]:
    """Outputs produced at or before stage x that a later stage reads."""
    before = [n for st in stage_nodes[:x + 1] for n in st]
    after = {n for st in stage_nodes[x + 1:] for n in st}
    return [u for u in before if any(u in _inputs(v, dims) for v in after)]


class RefPipeline:
    """The oracle's stages, built once (parameter copies, Adam state), so a
    timed caller measures `train` alone."""

    def __init__(self, dims: dict, init: Dict[str, torch.Tensor], stage_nodes: List[List[str]],
                 opt: dict, schedule: str = "async_1f1b", micro_batches: int = 0):
        self.l = len(stage_nodes)
        self.sync = schedule == "sync"
        self.stages = [RefStage(dims, init, nodes, opt, sync_m=micro_batches if self.sync else 0)
                       for nodes in stage_nodes]
        self.sends = [boundary(stage_nodes, x, dims) for x in range(self.l)]

    def train(self, ids: torch.Tensor, labels: torch.Tensor, steps: int = 1) -> List[List[float]]:
        """`steps` iterations of m micro-batches (ids/labels: int [m, b*s]) in
        the schedule's per-stage op order; returns the losses [steps][m]."""
        l, m, stages, sends = self.l, ids.shape[0], self.stages, self.sends
        if self.sync:
            assert all(st.sync_m == m for st in stages), "GPipe oracle built for another m"
        all_losses = []
        for _ in range(steps):
            losses = [0.0] * m
            if self.sync:
                ops = [[("fwd", j) for j in range(1, m + 1)] + [("bwd", j) for j in range(m, 0, -1)]
                       for _ in range(l)]
            else:
                ops = [one_f_one_b(l, m, x + 1) for x in range(l)]
            ptr = [0] * l
            acts: Dict[Tuple[int, int], Dict[str, torch.Tensor]] = {}
            grads: Dict[Tuple[int, int], Dict[str, torch.Tensor]] = {}
            left = sum(len(o) for o in ops)
            while left:
                moved = False
                for x in range(l):
                    while ptr[x] < len(ops[x]):
                        kind, j = ops[x][ptr[x]]
                        if kind == "fwd":
                            if x > 0 and (x - 1, j) not in acts:
                                break
                            recv = acts.get((x - 1, j), {})
                            env = stages[x].forward(j, recv, ids=ids[j - 1], labels=labels[j - 1])
                            fwd_env = dict(recv)
                            fwd_env.update(env)
                            if x < l - 1:
                                acts[(x, j)] = {u: fwd_env[u].detach() for u in sends[x]}
                            else:
                                losses[j - 1] = float(env["head"].detach())
                        else:
                            if x < l - 1 and (x, j) not in grads:
                                break
                            g_in = stages[x].backward(j, grads.pop((x, j), {}), sends[x])
                            if x > 0:
                                grads[(x - 1, j)] = g_in
                        ptr[x] += 1
                        left -= 1
                        moved = True
                if not moved:
                    raise RuntimeError("oracle schedule deadlock")
            for st in stages:
                st.flush()
            all_losses.append(losses)
        return all_losses

    def params(self) -> Dict[str, torch.Tensor]:
        final = {}
        for s in self.stages:
            final.update({k: v.detach().clone() for k, v in s.params.items()})
        return final


def reference_train(dims: dict, init: Dict[str, torch.Tensor], ids: torch.Tensor,
                    labels: torch.Tensor, stage_nodes: List[List[str]], opt: dict,
                    steps: int = 1, schedule: str = "async_1f1b"):
    """Run `steps` iterations of m micro-batches (ids/labels: int [m, b*s]).
    Returns (losses [steps][m], final fp32 parameters)."""
    ref = RefPipeline(dims, init, stage_nodes, opt, schedule, micro_batches=ids.shape[0])
    losses = ref.train(ids, labels, steps)
    return losses, ref.params()


def dims_from(cfg, nodes=None) -> dict:
    """The oracle's model description from a config object (attributes only) and,
    for CNN configs, the node structure (kind, inputs, geometry) as plain data."""
    d = dict(layers=cfg.layers, hidden=cfg.hidden, heads=cfg.heads, seq=cfg.seq, vocab=cfg.vocab,
             causal=cfg.causal, ln_eps=cfg.ln_eps, fused_attention=cfg.fused_attention,
             dec_layers=cfg.dec_layers, tgt_seq=cfg.tgt_seq)
    if getattr(cfg, "family", "transformer") == "cnn":
        d["graph"] = {n.id: (n.kind, tuple(n.inputs), dict(n.attrs)) for n in nodes}
    return d
