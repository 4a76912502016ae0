"""Per-stage device arenas: the stage's memory cap and its measured peak.

Each arena is one cudaMalloc of the stage's cap (`dpn_arena_create`).  torch's
caching allocator draws the stage's segments from it through a MemPool whose
pluggable allocator is the library's `dpn_arena_malloc` / `dpn_arena_free`
(include/dawnpiper.h): everything a stage allocates while its arena is active
-- weights, the weight-version ring, activation slots, transient tensors,
swap-in buffers, gradient buffers, kernel workspaces -- lives in the arena, so
an allocation past the cap fails like an out-of-memory on a GPU of that size,
and the arena's high-water mark is the stage's device peak (allocator
segments, fragmentation included).  This replaces the process-wide
`set_per_process_memory_fraction` cap for co-located stages: each stage has
its own cap, as on its own GPU.
"""

from __future__ import annotations

import ctypes as C
from contextlib import contextmanager
from typing import Tuple

import torch

from .._lib import SO_PATH, check, lib


class StageArena:
    def __init__(self, device: int, cap_bytes: int):
        h = C.c_int(-1)
        check(lib().dpn_arena_create(device, int(cap_bytes), C.byref(h)), "dpn_arena_create")
        self.handle = h.value
        self.device = device
        self._alloc = torch.cuda.memory.CUDAPluggableAllocator(
            str(SO_PATH), "dpn_arena_malloc", "dpn_arena_free")
        self.pool = torch.cuda.MemPool(self._alloc.allocator())

    @contextmanager
    def active(self):
        """Allocations on this thread go to this arena (through its MemPool)."""
        check(lib().dpn_arena_select(self.handle), "dpn_arena_select")
        try:
            with torch.cuda.use_mem_pool(self.pool, device=self.device):
                yield self
        finally:
            check(lib().dpn_arena_select(-1), "dpn_arena_select")

    def stats(self) -> Tuple[int, int, int]:
        """(bytes in use, high-water mark, capacity) of the arena."""
        used, peak, cap = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().dpn_arena_stats(self.handle, C.byref(used), C.byref(peak), C.byref(cap)),
              "dpn_arena_stats")
        return used.value, peak.value, cap.value

    def close(self) -> None:
        """Release the pool's segments back to the arena and the arena's
        reservation (every tensor allocated from it must be gone)."""
        import gc
        if self.pool is None:
            return
        self.pool = None
        self._alloc = None
        gc.collect()
        torch.cuda.synchronize(self.device)
        torch.cuda.empty_cache()
        # a block still referenced elsewhere (e.g. a cached workspace) keeps the
        # arena's reservation alive; the memory is returned by dpn_destroy
        lib().dpn_arena_destroy(self.handle)

    def reset_peak(self) -> None:
        check(lib().dpn_arena_reset_peak(self.handle), "dpn_arena_reset_peak")
