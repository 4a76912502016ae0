"""Per-stage device arenas (runtime/arena.py, dpn_arena_*): each co-located
stage allocates from its own cap-sized arena through a torch MemPool; the run
trains exactly as without arenas, the report's per-stage peaks are the arena
high-water marks, and a stage that outgrows its cap fails with an OOM."""
import pytest
import torch

from test_pipeline_gpu import _setup

pytestmark = pytest.mark.gpu


def _losses(cfg, g, plan, **kw):
    from paper_2505_05856_b200.runtime.model import AdamWConfig, synthetic_batch
    from paper_2505_05856_b200.runtime.pipeline import RunConfig, run
    rc = RunConfig(micro_batches=6, micro_batch_size=2, opt=AdamWConfig(lr=1e-3), **kw)
    ids, labels = synthetic_batch(cfg, 6, 2, seed=3)
    return run(plan, g, rc, model=cfg, ids=ids, labels=labels, steps=2)


def test_arenas_train_identically_and_measure_peaks():
    cfg, g, plan = _setup("tiny", 3, 0.6, 16 << 30)
    assert any(m.actions for m in plan.memopt)
    ref = _losses(cfg, g, plan)
    got = _losses(cfg, g, plan, capacity=2 << 30, arenas=True)
    assert got.per_stage_peak_source.startswith("measured")
    assert len(got.per_stage_peak) == 3 and all(0 < p <= 2 << 30 for p in got.per_stage_peak)
    for a, b in zip(got.losses, ref.losses):
        assert abs(a - b) <= 1e-3 * abs(b)


def test_arena_cap_raises_out_of_memory():
    cfg, g, plan = _setup("tiny", 2, 4.0, 16 << 30)
    with pytest.raises(torch.OutOfMemoryError):
        _losses(cfg, g, plan, capacity=1 << 20, arenas=True)


def test_arena_alloc_free_and_destroy():
    from paper_2505_05856_b200.runtime.arena import StageArena
    a = StageArena(0, 64 << 20)
    with a.active():
        x = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
        y = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
    used, peak, cap = a.stats()
    assert cap >= 64 << 20 and peak >= 16 << 20 and used >= 16 << 20
    del x, y
    torch.cuda.synchronize()
