"""B200 profiler: measured per-node times -> schema-1 profile graph.

The paper profiles each fine-grained op with timing hooks averaged over 50
iterations after warm-up and derives memory from the tensors the op
materialises.  Here one single-stage executor holds the
whole model; every node's forward and backward (as the executor actually runs
them, fusions included) is bracketed with CUDA events on the compute stream
for `iters` iterations after `warmup`, and the means become t_f / t_b in
integer microseconds.  Memory fields are exact byte counts of the executor's
tensors (runtime/graph.py).  The result loads in the reference's
`load_profile` unchanged and feeds `plan()`.
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple, Union

import torch

from .._lib import init_device
from ..planner.memplan import MemOptPlan
from ..planner.profile import ComputationGraph
from .graph import profile_graph
from .model import PRESETS, AdamWConfig, TransformerConfig, build_nodes, init_params, synthetic_batch
from .stage import StageExecutor


def measure_node_times(model: TransformerConfig, micro_batch: int, device: int = 0,
                       iters: int = 50, warmup: int = 5) -> Dict[str, Tuple[int, int]]:
    init_device(device)
    dev = torch.device("cuda", device)
    g0 = profile_graph(model, micro_batch)  # structure only (analytic times)
    nodes = build_nodes(model)
    stream = torch.cuda.Stream(device=dev)
    ex = StageExecutor(cfg=model, g=g0, nodes=nodes, lo=0, hi=len(nodes) - 1, stage=1, stages=1,
                       micro_batch=micro_batch, memopt=MemOptPlan(), init=init_params(model, 0),
                       device=dev, stream=stream, opt=AdamWConfig())
    ids, labels = synthetic_batch(model, 1, micro_batch, seed=0)
    ids, labels = ids.to(dev), labels.to(dev)
    loss = torch.zeros(1, device=dev)
    sums: Dict[Tuple[str, str], float] = {}
    torch.cuda.synchronize(dev)
    for it in range(warmup + iters):
        rec = it >= warmup
        ex.node_timer = [] if rec else None
        ex.forward(1, ids=ids[0], labels=labels[0], loss_out=loss)
        ex.backward(1)
        ex.finish_backward(1)
        if rec:
            torch.cuda.synchronize(dev)
            for nid, kind, e0, e1 in ex.node_timer:
                sums[(nid, kind)] = sums.get((nid, kind), 0.0) + e0.elapsed_time(e1)
    ex.node_timer = None
    out = {}
    for n in nodes:
        tf = sums.get((n.id, "fwd"), 0.0) / iters * 1000.0
        tb = sums.get((n.id, "bwd"), 0.0) / iters * 1000.0
        out[n.id] = (max(0, int(round(tf))), max(0, int(round(tb))))
    return out


def profile(model: Union[str, TransformerConfig], micro_batch: int, device: int = 0,
            iters: int = 50, warmup: int = 5) -> ComputationGraph:
    """Measured B200 profile of `model` at micro-batch size `micro_batch`."""
    cfg = PRESETS[model] if isinstance(model, str) else model
    times = measure_node_times(cfg, micro_batch, device, iters, warmup)
    return profile_graph(cfg, micro_batch, times=times, name=f"{cfg.name}_b{micro_batch}")
