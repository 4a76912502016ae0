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

Encoder-decoder (T5-large, BASELINE.json configs[3]): the encoder stack above
(non-causal, src tokens) ends in `enc_ln` = E; the decoder embeds the target
tokens (`dembed`) and runs blocks d{i} = causal self-attention sub-block,
cross-attention sub-block, FFN sub-block:
    c = lnx(y); q = c Wq^T + bq; kv = E Wkv^T + bkv; P = softmax(q K^T/sqrt(d));
    ctx = P V (node `xattn`: projections + fused cross-attention, q / kv / LSE
    saved inside it); y2 = ctx Wo^T + bo + y
then `lnf` and `head` over the target tokens.  The cross-attention is one
node (its K/V projection reads E) so that, in the reference's canonical order
(depth, fwd_start, id; graph.py:133), the K/V projections stay with their
layer and only E is relayed across decoder stages.  Node lists are returned
in canonical order (stable sort by depth), which for the decoder places the
target embedding and layer 0's self-attention sub-block beside the first
encoder layer, exactly where the reference planner would put them.
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
    # encoder-decoder: decoder layers and target length (0 = encoder / decoder only)
    dec_layers: int = 0
    tgt_seq: int = 0

    @property
    def encdec(self) -> bool:
        return self.dec_layers > 0

    @property
    def in_tokens(self) -> int:
        """Input token ids per sample (src, then tgt for encoder-decoder)."""
        return self.seq + self.tgt_seq

    @property
    def out_tokens(self) -> int:
        """Tokens per sample the head / loss runs over."""
        return self.tgt_seq if self.encdec else self.seq

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    family = "transformer"

    def input_spec(self, b: int):
        """Per-micro-batch input buffer: token ids int32 [b * in_tokens]."""
        return (b * self.in_tokens,), torch.int32

    @property
    def vocab_padded(self) -> int:
        # logits/head rows padded to a multiple of 64: 16-byte TMA strides and
        # full MMA tiles; the pad columns are masked out of the loss
        return (self.vocab + 63) // 64 * 64

    def n_params(self) -> int:
        H, F = self.hidden, self.ffn
        per_block = 4 * H + (3 * H * H + 3 * H) + (H * H + H) + (F * H + F) + (H * F + H)
        n = (self.vocab * H + self.seq * H + self.layers * per_block + 2 * H
             + self.vocab_padded * H)
        if self.encdec:
            cross = 2 * H + (H * H + H) + (2 * H * H + 2 * H) + (H * H + H)
            n += self.vocab * H + self.tgt_seq * H + self.dec_layers * (per_block + cross) + 2 * H
        return n

    def flops_per_sample(self) -> int:
        """Algorithmic training FLOPs per sample (3x forward; recompute excluded)."""
        H, F, s, L = self.hidden, self.ffn, self.seq, self.layers
        gemm = 2 * s * (3 * H * H + H * H + 2 * H * F) * L
        attn = 2 * 2 * s * s * H * L
        if self.encdec:
            t, D = self.tgt_seq, self.dec_layers
            gemm += 2 * t * (3 * H * H + H * H + 2 * H * F) * D      # self-attn + FFN
            gemm += 2 * (t * H * H + s * 2 * H * H + t * H * H) * D   # q, kv, out projections
            attn += 2 * 2 * t * t * H * D + 2 * 2 * t * s * H * D     # self + cross products
        head = 2 * self.out_tokens * H * self.vocab
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
    # BASELINE.json configs[3]: T5-large, 24 + 24 layers, d 1024, d_ff 4096, 16 heads,
    # vocab 32128; src 512 / tgt 128 (pinned here: BASELINE.json leaves seq open)
    "t5-large": TransformerConfig("t5-large", 24, 1024, 16, 4096, 32128, 512, dec_layers=24,
                                  tgt_seq=128),
    "tiny-t5": TransformerConfig("tiny-t5", 2, 128, 2, 256, 512, 128, dec_layers=2, tgt_seq=64),
}


@dataclass(frozen=True)
class NodeDef:
    id: str
    kind: str
    inputs: Tuple[str, ...]          # forward data inputs (node ids)
    params: Tuple[Tuple[str, Tuple[int, ...]], ...] = ()
    layer: int = -1
    seq: int = 0          # token rows per sample of this node's output
    causal: bool = False  # attention nodes: causal mask
    attrs: Tuple[Tuple[str, int], ...] = ()  # CNN nodes: spatial geometry (runtime/cnn.py)


def _ln(nid: str, x: str, H: int, layer: int, seq: int) -> NodeDef:
    return NodeDef(nid, "ln", (x,), (("gamma", (H,)), ("beta", (H,))), layer, seq)


def _block(cfg: TransformerConfig, p: str, x: str, layer: int, seq: int, causal: bool,
           cross_src: str = "") -> List[NodeDef]:
    """One pre-LN block; with cross_src, a cross-attention sub-block over that
    node's output sits between self-attention and the FFN (decoder block)."""
    H, F = cfg.hidden, cfg.ffn
    nodes = [_ln(p + "ln1", x, H, layer, seq),
             NodeDef(p + "qkv", "linear", (p + "ln1",), (("weight", (3 * H, H)), ("bias", (3 * H,))),
                     layer, seq)]
    if cfg.fused_attention:
        nodes.append(NodeDef(p + "attn", "attn_fused", (p + "qkv",), (), layer, seq, causal))
    else:
        nodes += [NodeDef(p + "score", "score", (p + "qkv",), (), layer, seq, causal),
                  NodeDef(p + "attn", "attn", (p + "score", p + "qkv"), (), layer, seq, causal)]
    nodes.append(NodeDef(p + "proj", "linear_res", (p + "attn", x),
                         (("weight", (H, H)), ("bias", (H,))), layer, seq))
    y = p + "proj"
    if cross_src:
        nodes += [
            _ln(p + "lnx", y, H, layer, seq),
            NodeDef(p + "xattn", "xattn", (p + "lnx", cross_src),
                    (("q_weight", (H, H)), ("q_bias", (H,)), ("kv_weight", (2 * H, H)),
                     ("kv_bias", (2 * H,))), layer, seq),
            NodeDef(p + "xproj", "linear_res", (p + "xattn", y), (("weight", (H, H)), ("bias", (H,))),
                    layer, seq),
        ]
        y = p + "xproj"
    nodes += [
        _ln(p + "ln2", y, H, layer, seq),
        NodeDef(p + "fc1", "linear", (p + "ln2",), (("weight", (F, H)), ("bias", (F,))), layer, seq),
        NodeDef(p + "gelu", "gelu", (p + "fc1",), (), layer, seq),
        NodeDef(p + "fc2", "linear", (p + "gelu",), (("weight", (H, F)), ("bias", (H,))), layer, seq),
        NodeDef(p + "add", "add", (p + "fc2", y), (), layer, seq),
    ]
    return nodes


def canonical_order(nodes: List[NodeDef]) -> List[NodeDef]:
    """Stable sort of a topological node list by depth (longest path from a
    source): the reference's canonical order (depth, fwd_start, id), graph.py:133,
    when fwd_start follows this list."""
    depth: Dict[str, int] = {}
    for n in nodes:
        depth[n.id] = max((depth[u] + 1 for u in n.inputs), default=0)
    return sorted(nodes, key=lambda n: depth[n.id])


def _cnn(cfg) -> bool:
    return getattr(cfg, "family", "transformer") == "cnn"


def build_nodes(cfg: TransformerConfig) -> List[NodeDef]:
    if _cnn(cfg):
        from . import cnn
        return cnn.build_nodes(cfg)
    H, Vp, S = cfg.hidden, cfg.vocab_padded, cfg.seq
    nodes = [NodeDef("embed", "embed", (), (("tok", (cfg.vocab, H)), ("pos", (S, H))), -1, S)]
    x = "embed"
    for b in range(cfg.layers):
        nodes += _block(cfg, f"b{b}.", x, b, S, cfg.causal and not cfg.encdec)
        x = f"b{b}.add"
    if cfg.encdec:
        T = cfg.tgt_seq
        nodes.append(_ln("enc_ln", x, H, -1, S))
        nodes.append(NodeDef("dembed", "embed", (), (("tok", (cfg.vocab, H)), ("pos", (T, H))), -1, T))
        x = "dembed"
        for b in range(cfg.dec_layers):
            nodes += _block(cfg, f"d{b}.", x, cfg.layers + b, T, True, cross_src="enc_ln")
            x = f"d{b}.add"
        S = T
    nodes.append(_ln("lnf", x, H, -1, S))
    nodes.append(NodeDef("head", "head", ("lnf",), (("weight", (Vp, H)),), -1, S))
    return canonical_order(nodes)


def node_rows(cfg: TransformerConfig, node: NodeDef, b: int) -> int:
    if _cnn(cfg):
        from . import cnn
        return cnn.node_rows(cfg, node, b)
    return b * (node.seq or cfg.seq)


def output_spec(cfg: TransformerConfig, node: NodeDef, b: int) -> Tuple[Tuple[int, ...], torch.dtype]:
    """Shape/dtype of a node's forward output for micro-batch size b."""
    if _cnn(cfg):
        from . import cnn
        return cnn.output_spec(cfg, node, b)
    M, H = node_rows(cfg, node, b), cfg.hidden
    k = node.kind
    if k in ("embed", "ln", "attn", "attn_fused", "linear_res", "add", "xattn"):
        return (M, H), torch.bfloat16
    if k == "linear":
        return (M, dict(node.params)["weight"][0]), torch.bfloat16
    if k == "gelu":
        return (M, cfg.ffn), torch.bfloat16
    if k == "score":
        s = node.seq or cfg.seq
        return (b, cfg.heads, s, s), torch.bfloat16
    if k == "head":  # saved dlogits (computed by the fused forward loss)
        return (M, cfg.vocab_padded), torch.bfloat16
    raise ValueError(k)


def internal_specs(cfg: TransformerConfig, node: NodeDef, b: int):
    """Tensors a node saves for its own backward besides its output and
    statistics: the cross-attention's q [b*t, H], kv [b*s, 2H] and P [b, A, t, s];
    max pooling's argmax taps."""
    if _cnn(cfg):
        from . import cnn
        return cnn.internal_specs(cfg, node, b)
    if node.kind != "xattn":
        return {}
    t, s, H = node.seq, cfg.seq, cfg.hidden
    out = {"q": ((b * t, H), torch.bfloat16), "kv": ((b * s, 2 * H), torch.bfloat16)}
    if cfg.fused_attention:  # flash-style kernel: only the per-row log-sum-exp is kept
        out["lse"] = ((b, cfg.heads, t), torch.float32)
    else:                    # materialised probabilities (reference vocabulary)
        out["p"] = ((b, cfg.heads, t, s), torch.bfloat16)
    return out


def stats_bytes(cfg: TransformerConfig, node: NodeDef, b: int) -> int:
    """Side statistics saved next to the output: LayerNorm (mean, rstd) per row,
    fused attention's log-sum-exp per (batch, head, query); batch-norm column
    sums (sum, sum of squares); fp32."""
    if _cnn(cfg):
        from . import cnn
        return cnn.stats_bytes(cfg, node, b)
    if node.kind == "ln":
        return 8 * node_rows(cfg, node, b)
    if node.kind == "attn_fused":
        return 4 * b * cfg.heads * (node.seq or cfg.seq)
    return 0


def has_stats(node: NodeDef) -> bool:
    return node.kind in ("ln", "attn_fused", "bn")


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
        elif n.kind == "xattn":
            readers[n.inputs[0]].append(n.id)         # c for the q-projection wgrad
            readers[n.inputs[1]].append(n.id)         # E for the kv-projection wgrad
            readers[n.id].append(n.id)                # O for D = rowsum(dO * O) (fused kernel)
            # (q, kv and P are internal tensors of the node itself)
        elif n.kind in ("bn", "pw", "dw"):
            readers[n.inputs[0]].append(n.id)         # x for BN's xhat / the weight gradients
        elif n.kind == "relu":
            readers[n.id].append(n.id)                # mask from the saved output
        # stem (reads the input images), pool (max: own argmax), add, concat,
        # gap: no saved activations
    # (LayerNorm statistics are a separate tensor, read only by their own node)
    return readers


def param_shapes(cfg: TransformerConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    if _cnn(cfg):
        from . import cnn
        return cnn.param_shapes(cfg)
    return [(f"{n.id}.{pn}", shp) for n in build_nodes(cfg) for pn, shp in n.params]


def init_params(cfg: TransformerConfig, seed: int = 0) -> Dict[str, torch.Tensor]:
    """Deterministic fp32 CPU initialisation shared by the B200 run and the
    CPU oracle: N(0, 0.02) matrices/embeddings, zero biases, LN (1, 0);
    head pad rows zero."""
    if _cnn(cfg):
        from . import cnn
        return cnn.init_params(cfg, seed)
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
    """Token ids int32 [m, b*in_tokens] (encoder-decoder: the b*s source ids,
    then the b*t target ids) and labels int32 [m, b*out_tokens], uniform over
    the vocabulary."""
    if _cnn(cfg):
        from . import cnn
        return cnn.synthetic_batch(cfg, micro_batches, b, seed)
    g = torch.Generator().manual_seed(seed + 1)
    ids = torch.randint(0, cfg.vocab, (micro_batches, b * cfg.in_tokens), generator=g,
                        dtype=torch.int64)
    labels = torch.randint(0, cfg.vocab, (micro_batches, b * cfg.out_tokens), generator=g,
                           dtype=torch.int64)
    return ids.to(torch.int32), labels.to(torch.int32)


@dataclass(frozen=True)
class AdamWConfig:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01


from .cnn import CNN_PRESETS, CNNConfig  # noqa: E402  (cnn.py imports NodeDef from here)

PRESETS.update(CNN_PRESETS)
