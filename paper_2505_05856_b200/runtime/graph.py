"""From a model config to the schema-1 profile graph the planner consumes.

`profile_graph(cfg, b, times)` produces exactly the reference data model
(`dawnplan/graph.py:55-89`): one ProfiledNode per executor node with
  * t_f / t_b   measured per-node B200 times in us (runtime/profiler.py), or an
                analytic estimate when no measurement is supplied;
  * m_a         bytes the node materialises (its output, plus LN statistics);
  * m_p         bytes of one bf16 weight version (what 1F1B weight stashing
                replicates l-x+1 times, matching schedule_weight);
  * m_d         bytes of un-saved tensors whose last forward reader is this node
                (e.g. fc2's output, freed once `add` has consumed it);
  * saved       the tensors some backward reads, with last_backward_access =
                the lowest-index backward reader (backward runs right to left).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import torch

from ..planner.profile import ComputationGraph, ProfiledNode, TensorRef
from .model import (NodeDef, TransformerConfig, backward_readers, build_nodes, has_stats,
                    internal_specs, node_rows, output_spec, saved_for_backward, stats_bytes)


def tensor_bytes(shape, dtype) -> int:
    n = 1
    for s in shape:
        n *= s
    return n * torch.empty((), dtype=dtype).element_size()


def out_tid(node_id: str) -> str:
    return f"{node_id}.out"


def stats_tid(node_id: str) -> str:
    return f"{node_id}.stats"


def internal_tid(node_id: str, name: str) -> str:
    return f"{node_id}.{name}"


def node_param_bytes(node: NodeDef) -> int:
    total = 0
    for _, shp in node.params:
        n = 1
        for s in shp:
            n *= s
        total += 2 * n
    return total


def analytic_times(cfg: TransformerConfig, b: int, tflops: float = 900.0,
                   gbs: float = 5000.0) -> Dict[str, Tuple[int, int]]:
    """Roofline estimate (us) per node: max(flops / tflops, bytes / gbs), bwd = 2x
    contraction work.  Only a placeholder until profiler times exist."""
    out = {}
    H = cfg.hidden
    for n in build_nodes(cfg):
        M, s = node_rows(cfg, n, b), n.seq or cfg.seq
        shape, dt = output_spec(cfg, n, b)
        byt = tensor_bytes(shape, dt)
        fl = 0
        if n.kind in ("linear", "linear_res", "head", "pw", "stem"):
            w = dict(n.params)["weight"]
            fl = 2 * M * w[0] * w[1]
        elif n.kind == "dw":
            fl = 2 * M * shape[1] * 9
        elif n.kind in ("score", "attn"):
            fl = 2 * b * cfg.heads * s * s * cfg.head_dim
        elif n.kind == "attn_fused":
            fl = 4 * b * cfg.heads * s * s * cfg.head_dim
        elif n.kind == "xattn":  # q and kv projections + the two attention products
            fl = 2 * M * H * H + 2 * b * cfg.seq * 2 * H * H + 4 * b * cfg.heads * s * cfg.seq * cfg.head_dim
        tf = max(1, int(round(max(fl / (tflops * 1e6), 2 * byt / (gbs * 1e3)))))
        tb = max(1, int(round(max(2 * fl / (tflops * 1e6), 3 * byt / (gbs * 1e3)))))
        out[n.id] = (tf, tb)
    return out


def profile_graph(cfg: TransformerConfig, b: int,
                  times: Optional[Dict[str, Tuple[int, int]]] = None,
                  name: Optional[str] = None) -> ComputationGraph:
    nodes = build_nodes(cfg)
    times = times or analytic_times(cfg, b)
    index = {n.id: i for i, n in enumerate(nodes)}
    consumers: Dict[str, List[str]] = {n.id: [] for n in nodes}
    for n in nodes:
        for u in n.inputs:
            consumers[u].append(n.id)
    readers = backward_readers(nodes)

    # depth = longest path over the consumer relation (graph.py:307-337)
    depth = {}
    for n in nodes:  # nodes are listed in a topological order
        depth[n.id] = max((depth[u] + 1 for u in n.inputs), default=0)

    # forward release: un-saved outputs die after their last forward reader
    release: Dict[str, int] = {n.id: 0 for n in nodes}
    for n in nodes:
        if not saved_for_backward(n) and consumers[n.id]:
            last = max(consumers[n.id], key=lambda c: index[c])
            shape, dt = output_spec(cfg, n, b)
            release[last] += tensor_bytes(shape, dt)

    out: List[ProfiledNode] = []
    clock = 0
    for i, n in enumerate(nodes):
        shape, dt = output_spec(cfg, n, b)
        internal = internal_specs(cfg, n, b)
        m_a = (tensor_bytes(shape, dt) + stats_bytes(cfg, n, b)
               + sum(tensor_bytes(shp, t) for shp, t in internal.values()))
        saved = []
        if saved_for_backward(n):
            rd = [index[r] for r in readers[n.id]]
            if rd:
                saved.append(TensorRef(out_tid(n.id), tensor_bytes(shape, dt), n.id, min(rd)))
        if has_stats(n):
            saved.append(TensorRef(stats_tid(n.id), stats_bytes(cfg, n, b), n.id, i))
        for nm, (shp, t) in internal.items():
            saved.append(TensorRef(internal_tid(n.id, nm), tensor_bytes(shp, t), n.id, i))
        t_f, t_b = times[n.id]
        out.append(ProfiledNode(
            id=n.id, depth=depth[n.id], fwd_start=clock, t_f=int(t_f), t_b=int(t_b), m_a=m_a,
            m_p=node_param_bytes(n), m_d=release[n.id], saved=tuple(saved),
            consumers=tuple(consumers[n.id])))
        clock += int(t_f)
    return ComputationGraph.build(name or f"{cfg.name}_b{b}", out)
