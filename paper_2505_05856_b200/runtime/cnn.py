"""AmoebaNet-D as a fine-grained node graph (BASELINE.json configs[4]).

The reference profiles CNNs with a conv / act / pool vocabulary
(`dawnplan/synth.py:111-155`); this is the executable counterpart.  Layout:
NHWC bf16 activations viewed as [pixels, channels].

Network (224x224x3 input, channels padded to 8 for 16-byte rows):
    stem   3x3 stride-2 convolution (im2col + tcgen05 GEMM) -> BN      112x112
    R0, R1 reduction cells                                              56, 28
    N normal cells, R2, N normal cells, R3, N normal cells              28, 14, 7
    head   ReLU -> global average pool -> FC (classes) -> cross entropy
Cells (NASNet / AmoebaNet form): inputs s0 (two cells back) and s1 (previous
cell) are preprocessed to the cell width F by ReLU -> 1x1 conv -> BN (s0 first
average-pooled with stride 2 when its resolution is twice s1's); five combine
steps each add two operations over earlier states; the cell output
concatenates three of the step outputs (3F channels).  Operations:
    sep3  ReLU -> depthwise 3x3 (stride s) -> 1x1 conv -> BN
    max3 / avg3   3x3 pooling (stride s; average excludes padding)
    id    identity (normal cells only)
In reduction cells the operations that read s0 / s1 use stride 2.  The
genotype below is an AmoebaNet-D-style cell of these operation types (the
published genotype also has 1x7-7x1 and 5x5 / 7x7 separable convolutions;
this build keeps the 3x3 family, stated in DESIGN.md).  Widths double at each
reduction, so memory is front-heavy and compute back-heavy -- the uneven
profile the planner is evaluated on.

Every 1x1 convolution is a GEMM over the [pixels, channels] view (no im2col);
depthwise convolutions, BN, ReLU, pooling and concat are HBM-bound kernels
(csrc/cnn.cu).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

import torch


IN_CH = 8  # input channels padded 3 -> 8 (16-byte pixel rows)

# (op_a, input_a, op_b, input_b) per step; inputs index [s0, s1, step0, step1, ...]
NORMAL = (("max3", 0, "sep3", 1), ("avg3", 1, "id", 0), ("sep3", 0, "avg3", 2),
          ("sep3", 3, "id", 1), ("avg3", 4, "sep3", 2))
NORMAL_CONCAT = (4, 5, 6)
REDUCE = (("max3", 0, "sep3", 1), ("avg3", 1, "sep3", 0), ("max3", 1, "sep3", 2),
          ("sep3", 3, "avg3", 2), ("max3", 4, "sep3", 5))
REDUCE_CONCAT = (4, 5, 6)


@dataclass(frozen=True)
class CNNConfig:
    name: str
    normal_cells: int     # N per stack
    filters: int          # F: cell width of the first normal stack
    image: int = 224
    classes: int = 1000
    stem_ch: int = 32
    bn_eps: float = 1e-5
    family: str = "cnn"

    # executor / pipeline interface shared with TransformerConfig
    @property
    def seq(self) -> int:          # input rows (pixels) per sample
        return self.image * self.image

    @property
    def in_tokens(self) -> int:
        return self.seq

    @property
    def out_tokens(self) -> int:   # loss rows per sample
        return 1

    @property
    def vocab(self) -> int:
        return self.classes

    @property
    def vocab_padded(self) -> int:
        return (self.classes + 63) // 64 * 64

    @property
    def encdec(self) -> bool:
        return False

    hidden = 0
    heads = 1
    head_dim = 0
    causal = False
    fused_attention = True
    dec_layers = 0
    tgt_seq = 0
    layers = 0

    @property
    def ln_eps(self) -> float:
        return self.bn_eps

    def input_spec(self, b: int):
        return (b * self.seq, IN_CH), torch.bfloat16

    def n_params(self) -> int:
        return sum(_numel(s) for _, s in param_shapes(self))

    def flops_per_sample(self) -> int:
        """3x the forward multiply-adds of the GEMM-shaped work (stem, 1x1
        convolutions, head) plus the depthwise convolutions, per sample."""
        f = 0
        for n in build_nodes(self):
            a = dict(n.attrs)
            P = a["Ho"] * a["Wo"]
            if n.kind in ("pw", "stem"):
                w = dict(n.params)["weight"]
                f += 2 * P * w[0] * w[1]
            elif n.kind == "dw":
                f += 2 * P * a["C"] * 9
            elif n.kind == "head":
                f += 2 * self.vocab_padded * a["C"]
        return 3 * f


def _numel(shape) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


class _Builder:
    def __init__(self, cfg: CNNConfig):
        self.cfg = cfg
        self.nodes: list = []
        self.meta: Dict[str, Tuple[int, int, int]] = {}  # node id -> (H, W, C) of its output

    def add(self, nid, kind, inputs, params=(), C=None, stride=1, mode=-1, layer=-1):
        from .model import NodeDef  # model.py imports this module at its end
        H, W, Cin = self.meta[inputs[0]] if inputs else (self.cfg.image, self.cfg.image, IN_CH)
        Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
        Co = C if C is not None else Cin
        attrs = (("H", H), ("W", W), ("Cin", Cin), ("Ho", Ho), ("Wo", Wo), ("C", Co),
                 ("stride", stride), ("mode", mode))
        self.nodes.append(NodeDef(nid, kind, tuple(inputs), tuple(params), layer, 0, False, attrs))
        self.meta[nid] = (Ho, Wo, Co)
        return nid

    def relu_conv_bn(self, p, x, C, layer):
        cin = self.meta[x][2]
        r = self.add(p + "relu", "relu", (x,), layer=layer)
        c = self.add(p + "pw", "pw", (r,), (("weight", (C, cin)),), C=C, layer=layer)
        return self.add(p + "bn", "bn", (c,), (("gamma", (C,)), ("beta", (C,))), layer=layer)

    def sep3(self, p, x, stride, layer):
        C = self.meta[x][2]
        r = self.add(p + "relu", "relu", (x,), layer=layer)
        d = self.add(p + "dw", "dw", (r,), (("weight", (C, 9)),), stride=stride, layer=layer)
        c = self.add(p + "pw", "pw", (d,), (("weight", (C, C)),), layer=layer)
        return self.add(p + "bn", "bn", (c,), (("gamma", (C,)), ("beta", (C,))), layer=layer)

    def op(self, p, kind, x, stride, layer):
        if kind == "sep3":
            return self.sep3(p + "sep.", x, stride, layer)
        if kind in ("max3", "avg3"):
            return self.add(p + kind, "pool", (x,), stride=stride, mode=0 if kind == "max3" else 1,
                            layer=layer)
        if kind == "id":
            assert stride == 1, "identity cannot reduce"
            return x
        raise ValueError(kind)

    def cell(self, name, s0, s1, C, reduce, layer):
        p = f"{name}."
        if self.meta[s0][0] != self.meta[s1][0]:  # s0 at twice the resolution: subsample first
            s0 = self.add(p + "pre0.sub", "pool", (s0,), stride=2, mode=1, layer=layer)
        states = [self.relu_conv_bn(p + "pre0.", s0, C, layer),
                  self.relu_conv_bn(p + "pre1.", s1, C, layer)]
        geno, concat = (REDUCE, REDUCE_CONCAT) if reduce else (NORMAL, NORMAL_CONCAT)
        for i, (oa, ia, ob, ib) in enumerate(geno):
            sa = 2 if (reduce and ia < 2) else 1
            sb = 2 if (reduce and ib < 2) else 1
            a = self.op(f"{p}s{i}.a.", oa, states[ia], sa, layer)
            b_ = self.op(f"{p}s{i}.b.", ob, states[ib], sb, layer)
            states.append(self.add(f"{p}s{i}.add", "add", (a, b_), layer=layer))
        ins = tuple(states[k] for k in concat)
        return self.add(p + "cat", "concat", ins, C=sum(self.meta[t][2] for t in ins), layer=layer)


def build_nodes(cfg: CNNConfig) -> list:
    from .model import canonical_order
    bd = _Builder(cfg)
    F = cfg.filters
    stem = bd.add("stem", "stem", (), (("weight", (cfg.stem_ch, 9 * IN_CH)),), C=cfg.stem_ch, stride=2)
    x = bd.add("stem.bn", "bn", (stem,), (("gamma", (cfg.stem_ch,)), ("beta", (cfg.stem_ch,))))
    s0, s1 = x, x
    layer = 0
    plan = [("r0", F // 2, True), ("r1", F, True)]
    widths = [F, 2 * F, 4 * F]
    for st, C in enumerate(widths):
        plan += [(f"n{st}_{i}", C, False) for i in range(cfg.normal_cells)]
        if st < 2:
            plan.append((f"r{st + 2}", 2 * C, True))
    for name, C, red in plan:
        out = bd.cell(name, s0, s1, C, red, layer)
        s0, s1 = s1, out
        layer += 1
    r = bd.add("head.relu", "relu", (s1,))
    g = bd.add("gap", "gap", (r,))
    C = bd.meta[g][2]
    bd.add("head", "head", (g,), (("weight", (cfg.vocab_padded, C)),))
    return canonical_order(bd.nodes)


def attrs(node) -> Dict[str, int]:
    return dict(node.attrs)


def node_rows(cfg: CNNConfig, node, b: int) -> int:
    a = attrs(node)
    if node.kind in ("gap", "head"):
        return b
    return b * a["Ho"] * a["Wo"]


def output_spec(cfg: CNNConfig, node, b: int):
    a = attrs(node)
    if node.kind == "head":
        return (b, cfg.vocab_padded), torch.bfloat16
    return (node_rows(cfg, node, b), a["C"]), torch.bfloat16


def internal_specs(cfg: CNNConfig, node, b: int):
    if node.kind == "pool" and attrs(node)["mode"] == 0:
        return {"arg": ((node_rows(cfg, node, b), attrs(node)["C"]), torch.uint8)}
    return {}


def stats_bytes(cfg: CNNConfig, node, b: int) -> int:
    return 8 * attrs(node)["C"] if node.kind == "bn" else 0


def param_shapes(cfg: CNNConfig):
    return [(f"{n.id}.{pn}", shp) for n in build_nodes(cfg) for pn, shp in n.params]


def init_params(cfg: CNNConfig, seed: int = 0) -> Dict[str, torch.Tensor]:
    """He-normal convolutions (fan-in), depthwise N(0, 2/9), BN (1, 0), FC
    N(0, 0.01) with zero pad rows."""
    g = torch.Generator().manual_seed(seed)
    out: Dict[str, torch.Tensor] = {}
    for name, shp in param_shapes(cfg):
        pn = name.rsplit(".", 1)[1]
        if pn == "gamma":
            t = torch.ones(shp)
        elif pn == "beta":
            t = torch.zeros(shp)
        elif name == "head.weight":
            t = torch.randn(shp, generator=g) * 0.01
            t[cfg.classes:] = 0
        else:
            t = torch.randn(shp, generator=g) * (2.0 / shp[1]) ** 0.5
            if name == "stem.weight":  # padded input channels carry zeros: zero their taps too
                t.view(shp[0], 9, IN_CH)[:, :, 3:] = 0
        out[name] = t
    return out


def synthetic_batch(cfg: CNNConfig, micro_batches: int, b: int, seed: int = 0):
    """Images ~N(0, 1) as NHWC bf16 [m, b*H*W, 8] (channels 3..7 zero) and
    labels int32 [m, b] uniform over the classes."""
    g = torch.Generator().manual_seed(seed + 1)
    img = torch.zeros(micro_batches, b * cfg.seq, IN_CH)
    img[:, :, :3] = torch.randn(micro_batches, b * cfg.seq, 3, generator=g)
    labels = torch.randint(0, cfg.classes, (micro_batches, b), generator=g, dtype=torch.int64)
    return img.to(torch.bfloat16), labels.to(torch.int32)


CNN_PRESETS = {
    # BASELINE.json configs[4]: AmoebaNet-D at 224x224 (~28M parameters)
    # (N=5 normal cells per stack, F=144: 26.7M parameters)
    "amoebanet-d": CNNConfig("amoebanet-d", normal_cells=5, filters=144),
    # small shapes for parity tests
    "tiny-amoeba": CNNConfig("tiny-amoeba", normal_cells=1, filters=16, image=64, classes=10,
                             stem_ch=16),
}
