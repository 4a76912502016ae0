"""Debug helper: two stage processes on one GPU (gloo), checksums of boundary traffic."""
import os, sys, socket
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch
import torch.multiprocessing as mp


def worker(rank, port, name, stages):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=stages)
    import paper_2505_05856_b200.runtime.distributed as D
    from test_distributed_gpu import _plan
    from paper_2505_05856_b200 import planner as P
    from paper_2505_05856_b200._lib import init_device
    from paper_2505_05856_b200.runtime.model import AdamWConfig, build_nodes, init_params, synthetic_batch
    from paper_2505_05856_b200.runtime.stage import StageExecutor
    torch.cuda.set_device(0); init_device(0)
    cfg, g, plan = _plan(name, stages, 4.0, 16 << 30, 2)
    lo, hi = P.stage_bounds(plan.cuts, len(g))[rank]
    dev = torch.device("cuda", 0)
    st = StageExecutor(cfg=cfg, g=g, nodes=build_nodes(cfg), lo=lo, hi=hi, stage=rank + 1, stages=stages,
                       micro_batch=2, memopt=plan.memopt[rank], init=init_params(cfg, 0), device=dev,
                       stream=torch.cuda.Stream(dev), opt=AdamWConfig(lr=1e-3))
    print(rank, "recv", st.recv_ids, "send", st.send_ids, flush=True)
    os_send, os_recv = D.Wire.send, D.Wire.recv
    def send(self, t, dst, group):
        torch.cuda.synchronize(); print(f"r{rank} send {tuple(t.shape)} {t.dtype} sum={t.float().sum().item():.4f}", flush=True)
        return os_send(self, t, dst, group)
    D.Wire.send = send
    orig_adopt = st.adopt_recv
    def adopt(tid, j, t):
        torch.cuda.synchronize(); print(f"r{rank} adopt {tid} j={j} sum={t.float().sum().item():.4f}", flush=True)
        orig_adopt(tid, j, t)
    st.adopt_recv = adopt
    ids, labels = synthetic_batch(cfg, 3, 2, seed=3)
    loss = torch.zeros(3, device=dev)
    D.run_stage_step(st, D.BoundaryChannels(stages), rank, stages, 3, ids.to(dev) if st.needs_ids else None,
                     labels.to(dev) if st.is_last else None, loss if st.is_last else None)
    torch.cuda.synchronize()
    if st.is_last:
        print("losses", loss.tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    stages = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    ps = [ctx.Process(target=worker, args=(r, port, name, stages)) for r in range(stages)]
    [p.start() for p in ps]; [p.join(120) for p in ps]
    # co-located reference
    from paper_2505_05856_b200.runtime.pipeline import Pipeline, RunConfig
    from paper_2505_05856_b200.runtime.model import AdamWConfig, synthetic_batch
    from test_distributed_gpu import _plan
    cfg, g, plan = _plan(name, stages, 4.0, 16 << 30, 2)
    pipe = Pipeline(cfg, g, plan, RunConfig(micro_batches=3, micro_batch_size=2, opt=AdamWConfig(lr=1e-3), trace=False))
    ids, labels = synthetic_batch(cfg, 3, 2, seed=3)
    print("colocated losses", pipe.step(ids.cuda(), labels.cuda()).tolist())
