"""World-size-2/3 gloo runs of the per-stage 1F1B scheduler (runtime/distributed.py).

A stand-in stage does deterministic scalar work on CPU tensors; the test checks
that every rank runs exactly async_ops(l, m, x), that activations and gradients
arrive matched to the right micro-batch over the per-direction channels, and
that the run does not deadlock.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeStage:
    """y = x + 10*stage (+ ids for stage 1); grad in = grad out + stage."""

    def __init__(self, rank, world, stages=None):
        l = stages or world
        self.rank, self.world = rank, world
        self.replica = rank // l
        self.x = rank % l + 1
        self.is_first, self.is_last = self.x == 1, self.x == l
        self.recv_ids = [] if self.is_first else ["act"]
        self.send_ids = [] if self.is_last else ["act"]
        self.inbox = {}
        self.outbox = {}
        self.grads = {}
        self.log = []
        self.results = {}
        self.wgrad = torch.zeros(3)
        self.synced = []  # weight gradient seen by each optimizer update

    def recv_buffer(self, tid, j):
        self.inbox[j] = torch.zeros(4)
        return self.inbox[j]

    def send_buffer(self, tid, j):
        return self.outbox[j]

    def forward(self, j, ids=None, labels=None, loss_out=None):
        self.log.append(("fwd", j))
        x = ids.float() if self.is_first else self.inbox[j]
        y = x + 10 * self.x
        self.outbox[j] = y
        if self.is_last:
            self.results[j] = y.clone()

    def grad_like(self, tid):
        return torch.zeros(4)

    def set_recv_grad(self, tid, t):
        self.grads[tid] = t

    def backward(self, j):
        self.log.append(("bwd", j))
        self.wgrad += float((self.replica + 1) * j)  # replica-specific weight gradient
        g = self.grads.get("act", torch.full((4,), float(j)))  # last stage seeds with j
        return {"act": g + self.x}

    def dp_grads(self):
        return [self.wgrad]

    def finish_backward(self, j):
        self.grads = {}
        if not self.sync:
            self.synced.append(self.wgrad[0].item())
            self.wgrad.zero_()

    def optimizer_step(self):
        self.log.append(("opt", 0))
        self.synced.append(self.wgrad[0].item())


class OverlappedFakeStage(FakeStage):
    """FakeStage with the executor's zero-copy receive / send hooks, so the
    scheduler takes its overlapped protocol (early-posted receives adopted by
    the stage, sends from released buffers)."""

    def recv_like(self, tid):
        return torch.zeros(4)

    def adopt_recv(self, tid, j, t):
        self.inbox[j] = t

    def release_send_buffer(self, tid, j):
        return self.outbox.pop(j)

    def slot_of(self, j):
        return (j - 1) % (self.world - self.x + 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, q, schedule="async_1f1b", stages=None, overlapped=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_05856_b200.runtime.distributed import BoundaryChannels, run_stage_step
    from paper_2505_05856_b200.planner.schedule import async_ops, sync_ops
    chans = BoundaryChannels(world, stages)
    l = chans.stages
    st = (OverlappedFakeStage if overlapped else FakeStage)(rank, world, stages)
    st.sync = schedule == "sync"
    # replica k's ids are offset by 1000 k: a message crossing replicas shows up
    ids = (torch.arange(m * 4, dtype=torch.int32).reshape(m, 4) + 1000 * st.replica
           if st.is_first else None)
    grads_seen = {}
    orig_set = st.set_recv_grad

    def spy(tid, t, _o=orig_set):
        grads_seen[len(grads_seen) + 1] = t.clone()
        _o(tid, t)
    st.set_recv_grad = spy
    run_stage_step(st, chans, rank, world, m, ids=ids, schedule=schedule)
    if schedule == "sync":
        expect = [(k, j) for k, j, _ in sync_ops(l, m, st.x)] + [("opt", 0)]
    else:
        expect = [(k, j) for k, j, _ in async_ops(l, m, st.x)]
    q.put((rank, st.log == expect, {j: v.tolist() for j, v in st.results.items()},
           {k: v.tolist() for k, v in grads_seen.items()}, st.synced))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,schedule,overlapped",
                         [(2, 5, "async_1f1b", False), (3, 7, "async_1f1b", False),
                          (2, 4, "sync", False), (3, 5, "sync", False),
                          (3, 7, "async_1f1b", True), (3, 5, "sync", True)])
def test_gloo_pipeline_order_and_matching(world, m, schedule, overlapped):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q, schedule, None, overlapped))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, ok, res, grads, _ = q.get(timeout=120)
        out[rank] = (ok, res, grads)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert out[r][0], f"rank {r} did not run the {schedule} op order"
    # last stage output of micro-batch j: ids[j] + 10 * (1 + 2 + ... + world)
    res = out[world - 1][1]
    shift = 10 * sum(range(1, world + 1))
    for j in range(1, m + 1):
        assert res[j] == [float((j - 1) * 4 + i + shift) for i in range(4)]
    # gradients received by stage x (x < l), in backward order (1F1B: j = 1..m,
    # GPipe: j = m..1): seed j at the last stage, + x' added by every stage x' > x
    for r in range(world - 1):
        add = sum(range(r + 2, world + 1))
        grads = out[r][2]
        for k in range(1, m + 1):
            j = m + 1 - k if schedule == "sync" else k
            assert grads[k] == [float(j + add)] * 4


@pytest.mark.parametrize("world,stages,m,schedule", [(4, 2, 5, "async_1f1b"), (4, 2, 4, "sync"),
                                                     (6, 3, 5, "async_1f1b")])
def test_gloo_data_parallel_replicas(world, stages, m, schedule):
    """world = l * d: every replica runs its own pipeline on its own data, and
    every optimizer update sees the weight gradient summed over the replicas."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q, schedule, stages))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, ok, res, grads, synced = q.get(timeout=120)
        out[rank] = (ok, res, grads, synced)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = world // stages
    shift = 10 * sum(range(1, stages + 1))
    for r in range(world):
        k, x = r // stages, r % stages + 1
        assert out[r][0], f"rank {r} did not run the {schedule} op order"
        if x == stages:  # last stage of replica k: its own replica's ids only
            for j in range(1, m + 1):
                assert out[r][1][j] == [float((j - 1) * 4 + i + shift + 1000 * k) for i in range(4)]
        # replica k contributes (k+1)*j per backward; the all-reduce sums replicas
        rep_sum = sum(range(1, d + 1))
        if schedule == "sync":
            assert out[r][3] == [float(rep_sum * sum(range(1, m + 1)))]
        else:
            assert out[r][3] == [float(rep_sum * j) for j in range(1, m + 1)]


def test_replica_layout_rejects_ragged_world():
    """world must be a whole number of replicas of the stage plan."""
    from paper_2505_05856_b200.runtime.distributed import BoundaryChannels
    with pytest.raises(ValueError, match="multiple of the stage count"):
        BoundaryChannels(6, 4)  # raises before any process group is created
