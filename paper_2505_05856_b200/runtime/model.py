"""Transformer model families as fine-grained node graphs.

The node vocabulary follows the reference profile generator
(`dawnplan/synth.py:22-26,93-107`: embed, per-block ln1 q k v score attn proj
ln2 fc1 gelu fc2 add, head) with two B200-first changes, both stated in
DESIGN.md: q/k/v are one fused `qkv` GEMM node (one N=3H contraction instead
of three N=H ones that underfill 148 SMs), and the final LayerNorm is its own
`lnf` node before `head` (vocab projection + cross-entropy).

Block (pre-LN, residuals folded into the producing GEMM / add node):
    h1 = ln1(x); qkv = h1 Wqkv^T + b; P = softmax(QK^T/sqrt(d) [+causal]);
    ctx = P V; y = ctx Wo^T + bo + x; h2 = ln2(y); f = h2 W1^T + b1;
    g = gelu(f); z = g W2^T + b2; out = z + y
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import torch


@dataclass(frozen=True)
class TransformerConfig:
    name: str
    layers: int
    hidden: int
    heads: int
    ffn: int
    vocab: int
    seq: int
    causal: bool = False
    ln_eps: float = 1e-5
    # one fused flash-style `attn` node (QKV -> context, P never materialised)
    # instead of the reference vocabulary's `score` + `attn` pair
    fused_attention: bool = True

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def vocab_padded(self) -> int:
        # logits/head rows padded to a multiple of 64: 16-byte TMA strides and
        # full MMA tiles; the pad columns are masked out of the loss
        return (self.vocab + 63) // 64 * 64

    def n_params(self) -> int:
        H, F = self.hidden, self.ffn
        per_block = 4 * H + (3 * H * H + 3 * H) + (H * H + H) + (F * H + F) + (H * F + H)
        return (self.vocab * H + self.seq * H + self.layers * per_block + 2 * H
                + self.vocab_padded * H)

    def flops_per_sample(self) -> int:
        """Algorithmic training FLOPs per sample (3x forward; recompute excluded)."""
        H, F, s, L = self.hidden, self.ffn, self.seq, self.layers
        gemm = 2 * s * (3 * H * H + H * H + 2 * H * F) * L
        attn = 2 * 2 * s * s * H * L
        head = 2 * s * H * self.vocab
        return 3 * (gemm + attn + head)


PRESETS: Dict[str, TransformerConfig] = {
    # BASELINE.json configs[0]: BERT-base, seq 128 (the reference CPU run)
    "bert-base": TransformerConfig("bert-base", 12, 768, 12, 3072, 30522, 128),
    # BASELINE.json configs[1]: BERT-large, seq 512 (the bench workload)
    "bert-large": TransformerConfig("bert-large", 24, 1024, 16, 4096, 30522, 512),
    # BASELINE.json configs[2]: GPT-2 XL 1.5B, seq 1024, causal
    "gpt2-xl": TransformerConfig("gpt2-xl", 48, 1600, 25, 6400, 50257, 1024, causal=True),
    # small shapes for parity tests
    "tiny": TransformerConfig("tiny", 2, 128, 2, 512, 1000, 64),
    "tiny-causal": TransformerConfig("tiny-causal", 3, 128, 2, 256, 512, 128, causal=True),
    "tiny-unfused": TransformerConfig("tiny-unfused", 2, 128, 2, 512, 1000, 64, fused_attention=False),
}


@dataclass(frozen=True)
class NodeDef:
    id: str
    kind: str
    inputs: Tuple[str, ...]          # forward data inputs (node ids)
    params: Tuple[Tuple[str, Tuple[int, ...]], ...] = ()
    layer: int = -1


def build_nodes(cfg: TransformerConfig) -> List[NodeDef]:
    H, F, Vp = cfg.hidden, cfg.ffn, cfg.vocab_padded
    nodes = [NodeDef("embed", "embed", (), (("tok", (cfg.vocab, H)), ("pos", (cfg.seq, H))))]
    x = "embed"
    for b in range(cfg.layers):
        p = f"b{b}."
        nodes += [
            NodeDef(p + "ln1", "ln", (x,), (("gamma", (H,)), ("beta", (H,))), b),
            NodeDef(p + "qkv", "linear", (p + "ln1",), (("weight", (3 * H, H)), ("bias", (3 * H,))), b),
        ]
        if cfg.fused_attention:
            nodes.append(NodeDef(p + "attn", "attn_fused", (p + "qkv",), (), b))
        else:
            nodes += [NodeDef(p + "score", "score", (p + "qkv",), (), b),
                      NodeDef(p + "attn", "attn", (p + "score", p + "qkv"), (), b)]
        nodes += [
            NodeDef(p + "proj", "linear_res", (p + "attn", x), (("weight", (H, H)), ("bias", (H,))), b),
            NodeDef(p + "ln2", "ln", (p + "proj",), (("gamma", (H,)), ("beta", (H,))), b),
            NodeDef(p + "fc1", "linear", (p + "ln2",), (("weight", (F, H)), ("bias", (F,))), b),
            NodeDef(p + "gelu", "gelu", (p + "fc1",), (), b),
            NodeDef(p + "fc2", "linear", (p + "gelu",), (("weight", (H, F)), ("bias", (H,))), b),
            NodeDef(p + "add", "add", (p + "fc2", p + "proj"), (), b),
        ]
        x = p + "add"
    nodes.append(NodeDef("lnf", "ln", (x,), (("gamma", (H,)), ("beta", (H,)))))
    nodes.append(NodeDef("head", "head", ("lnf",), (("weight", (Vp, H)),)))
    return nodes


def output_spec(cfg: TransformerConfig, node: NodeDef, b: int) -> Tuple[Tuple[int, ...], torch.dtype]:
    """Shape/dtype of a node's forward output for micro-batch size b."""
    M, H = b * cfg.seq, cfg.hidden
    k = node.kind
    if k in ("embed", "ln", "attn", "attn_fused", "linear_res", "add"):
        return (M, H), torch.bfloat16
    if k == "linear":
        return (M, dict(node.params)["weight"][0]), torch.bfloat16
    if k == "gelu":
        return (M, cfg.ffn), torch.bfloat16
    if k == "score":
        return (b, cfg.heads, cfg.seq, cfg.seq), torch.bfloat16
    if k == "head":  # saved dlogits (computed by the fused forward loss)
        return (M, cfg.vocab_padded), torch.bfloat16
    raise ValueError(k)


def stats_bytes(cfg: TransformerConfig, node: NodeDef, b: int) -> int:
    """Side statistics saved next to the output: LayerNorm (mean, rstd) per row,
    fused attention's log-sum-exp per (batch, head, query); fp32."""
    if node.kind == "ln":
        return 8 * b * cfg.seq
    if node.kind == "attn_fused":
        return 4 * b * cfg.heads * cfg.seq
    return 0


def has_stats(node: NodeDef) -> bool:
    return node.kind in ("ln", "attn_fused")


def saved_for_backward(node: NodeDef) -> bool:
    """Whether some backward reads this node's output (fc2's z is only summed)."""
    return not (node.kind == "linear" and node.id.endswith(".fc2"))


def backward_readers(nodes: List[NodeDef]) -> Dict[str, List[str]]:
    """node id -> ids of nodes whose *backward* reads that node's output."""
    readers: Dict[str, List[str]] = {n.id: [] for n in nodes}
    for n in nodes:
        if n.kind in ("ln", "linear", "linear_res"):
            readers[n.inputs[0]].append(n.id)         # LN input x / GEMM input for wgrad
        elif n.kind == "head":
            readers[n.inputs[0]].append(n.id)         # wgrad reads lnf output
            readers[n.id].append(n.id)                # saved dlogits
        elif n.kind == "gelu":
            readers[n.inputs[0]].append(n.id)         # gelu'(f)
        elif n.kind == "score":
            readers[n.inputs[0]].append(n.id)         # Q, K for dQ, dK
            readers[n.id].append(n.id)                # P for the softmax backward
        elif n.kind == "attn":
            readers[n.inputs[0]].append(n.id)         # P for dV
            readers[n.inputs[1]].append(n.id)         # V for dP
        elif n.kind == "attn_fused":
            readers[n.inputs[0]].append(n.id)         # Q, K, V (S and P are recomputed)
            readers[n.id].append(n.id)                # O for D = rowsum(dO * O)
    # (LayerNorm statistics are a separate tensor, read only by their own node)
    return readers


def param_shapes(cfg: TransformerConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    return [(f"{n.id}.{pn}", shp) for n in build_nodes(cfg) for pn, shp in n.params]


def init_params(cfg: TransformerConfig, seed: int = 0) -> Dict[str, torch.Tensor]:
    """Deterministic fp32 CPU initialisation shared by the B200 run and the
    CPU oracle: N(0, 0.02) matrices/embeddings, zero biases, LN (1, 0);
    head pad rows zero."""
    g = torch.Generator().manual_seed(seed)
    out: Dict[str, torch.Tensor] = {}
    for name, shp in param_shapes(cfg):
        pn = name.rsplit(".", 1)[1]
        if pn == "gamma":
            t = torch.ones(shp)
        elif pn in ("beta", "bias"):
            t = torch.zeros(shp)
        else:
            t = torch.randn(shp, generator=g) * 0.02
            if name == "head.weight":
                t[cfg.vocab:] = 0
        out[name] = t
    return out


def synthetic_batch(cfg: TransformerConfig, micro_batches: int, b: int, seed: int = 0):
    """Token ids and labels, int32 [m, b*s], uniform over the vocabulary."""
    g = torch.Generator().manual_seed(seed + 1)
    ids = torch.randint(0, cfg.vocab, (micro_batches, b * cfg.seq), generator=g, dtype=torch.int64)
    labels = torch.randint(0, cfg.vocab, (micro_batches, b * cfg.seq), generator=g, dtype=torch.int64)
    return ids.to(torch.int32), labels.to(torch.int32)


@dataclass(frozen=True)
class AdamWConfig:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
