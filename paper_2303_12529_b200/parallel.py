"""Clip-parallel execution across GPUs (BASELINE configs[2]).

Independent clips are the unit of work: clip i runs on rank i mod world
(round robin), each rank owns its own device spectra, and no collective
touches the data path.  The only communication is the gather of the small
per-clip records at the end and the max-over-ranks of the timings, over
whatever `torch.distributed` backend the caller initialised (NCCL on the GPU
box, gloo in the CPU tests).

The reference has no multi-process code; its contract allows independent runs
to execute concurrently (`SPEC.md:432`), which is what this module does.
"""

from __future__ import annotations

import time
from dataclasses import asdict, dataclass


@dataclass
class ClipRecord:
    """Per-clip outcome of one solve (the fields of `MetricsReport`, metrics.py:16-31)."""
    index: int
    rank: int
    l2: int
    pvband: int
    shots: int
    iters: int
    wall_time: float


def world_info(group=None):
    """(rank, world size) of the default group, or (0, 1) without one."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard(n_items, rank, world):
    """Indices owned by `rank`: round robin, disjoint, covering 0..n_items-1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return list(range(rank, n_items, world))


def max_over_ranks(value, group=None, device=None):
    """Max of a float over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    if dist.get_backend(group) != "nccl":
        device = "cpu"  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_records(records, group=None):
    """All ranks' records, ordered by clip index (every rank gets the list)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return sorted(records, key=lambda r: r.index)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, [asdict(r) for r in records], group=group)
    merged = [ClipRecord(**d) for part in out for d in part]
    return sorted(merged, key=lambda r: r.index)


def optimize_batch(targets, focus_kernels, defocus_kernels, cfg, group=None, solver=None,
                   synchronize=None, lanes=2, results=None):
    """Solve every clip of `targets` (a sequence of 2-D uint8 layouts; a
    `LazyClips` lets each rank generate only its own clips) on the rank that
    owns it.  Returns (records of all clips ordered by index,
    seconds = max over ranks of this rank's solve time).

    `solver(target, focus, defocus, cfg) -> OptimizationResult` replaces the
    device loop (tests inject a stub).  Without it, `lanes` concurrent
    streams each solve every lanes-th clip of this rank's shard.  `results`
    (a dict, optional) receives this rank's OptimizationResult per clip index.
    """
    rank, world = world_info(group)
    mine = [(i, targets[i]) for i in shard(len(targets), rank, world)]  # inputs built before timing
    if synchronize:
        synchronize()
    t0 = time.perf_counter()
    records = []

    def record(i, r):
        if results is not None:
            results[i] = r
        m = r.metrics
        records.append(ClipRecord(i, rank, int(m.l2), int(m.pvband), int(m.shots), int(r.iters_run),
                                  float(r.wall_time)))

    if solver is not None:
        for i, target in mine:
            record(i, solver(target, focus_kernels, defocus_kernels, cfg))
    else:
        # `lanes` worker threads, each with its own CUDA stream and work
        # buffers (nv.set_lane), solve alternate clips: one lane's host-side
        # gaps (session set-up, stop-flag polls, copies, shot count) overlap
        # the other lane's device loop.
        import threading
        from concurrent.futures import ThreadPoolExecutor

        import torch

        from . import _native as nv
        from .optimizer import _assemble, _optimize_device
        lock = threading.Lock()
        dev = torch.cuda.current_device()

        def worker(lane, items):
            nv.set_lane(lane)
            torch.cuda.set_device(dev)
            stream = torch.cuda.Stream()
            # the shot count runs on a host tail thread; a clip is assembled
            # (waiting for its count) only after the lane's next clip has run,
            # so the count never stalls the lane
            pending = None

            def flush(p):
                r = _assemble(p[1], cfg)
                with lock:
                    record(p[0], r)

            with torch.cuda.stream(stream):
                for i, target in items:
                    parts = _optimize_device(target, focus_kernels, defocus_kernels, cfg, shots_on="host")
                    if pending is not None:
                        flush(pending)
                    pending = (i, parts)
            stream.synchronize()
            if pending is not None:
                flush(pending)

        with ThreadPoolExecutor(max_workers=lanes) as pool:
            for f in [pool.submit(worker, l, mine[l::lanes]) for l in range(lanes)]:
                f.result()
    if synchronize:
        synchronize()
    seconds = max_over_ranks(time.perf_counter() - t0, group)
    return gather_records(records, group), seconds


def modulation_search_sharded(phi_gt, target, focus_kernels, defocus_kernels, cfg, num_samples=41,
                              eval_steps=10, group=None, lanes=2, scorer=None, synchronize=None):
    """`modulation_search` (optimizer.py:294-341) with its candidates spread
    over the ranks: candidate i runs on rank i mod world,
    `lanes` streams per GPU score alternate candidates, and one all-gather of
    the (index, delta_h, L_DSO) triples gives every rank the full candidate
    list, from which each picks the same winner with the reference's
    tie-break.  Returns (ModulationSearchResult, seconds = max over ranks).

    `scorer(dh) -> L_DSO` replaces the device evaluation (tests inject a stub).
    """
    import torch.distributed as dist

    from .optimizer import (_check_target, modulation_eval_cfg, modulation_offsets, modulation_pick,
                            modulation_score)
    rank, world = world_info(group)
    offsets = modulation_offsets(num_samples)
    target = _check_target(target)
    eval_cfg = modulation_eval_cfg(cfg)
    mine = [(i, offsets[i]) for i in shard(len(offsets), rank, world)]
    if synchronize:
        synchronize()
    t0 = time.perf_counter()
    scored = []
    if scorer is not None:
        scored = [(i, dh, float(scorer(dh))) for i, dh in mine]
    else:
        import threading
        from concurrent.futures import ThreadPoolExecutor

        import torch

        from . import _native as nv
        lock = threading.Lock()
        dev = torch.cuda.current_device()

        def worker(lane, items):
            nv.set_lane(lane)
            torch.cuda.set_device(dev)
            stream = torch.cuda.Stream()
            resident = {}  # phi_gt and the target stay on the device for this lane's candidates
            with torch.cuda.stream(stream):
                for i, dh in items:
                    loss = modulation_score(phi_gt, target, focus_kernels, defocus_kernels, eval_cfg, dh, eval_steps,
                                            resident)
                    with lock:
                        scored.append((i, dh, loss))
            stream.synchronize()

        with ThreadPoolExecutor(max_workers=lanes) as pool:
            for f in [pool.submit(worker, l, mine[l::lanes]) for l in range(lanes)]:
                f.result()
    if synchronize:
        synchronize()
    seconds = max_over_ranks(time.perf_counter() - t0, group)
    if dist.is_available() and dist.is_initialized():
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, scored, group=group)
        scored = [t for part in parts for t in part]
    scored.sort(key=lambda t: t[0])
    if [t[0] for t in scored] != list(range(len(offsets))):
        raise RuntimeError("modulation_search_sharded: candidate set incomplete after the gather")
    # with a stub scorer (CPU tests) the winning gate is formed on the host
    gate = (lambda p: p >= 0.0) if scorer is not None else None
    return modulation_pick(phi_gt, [(dh, l) for _, dh, l in scored], gate), seconds


def warm_lanes(target, focus_kernels, defocus_kernels, cfg, lanes=2):
    """Solve `target` once on every lane (no collectives), so the lanes'
    spectra, work buffers and captured iteration graphs exist before timing."""
    import torch

    from . import _native as nv
    from .optimizer import optimize
    dev = torch.cuda.current_device()
    for lane in range(lanes):
        prev = nv.lane()
        nv.set_lane(lane)
        try:
            torch.cuda.set_device(dev)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                optimize(target, focus_kernels, defocus_kernels, cfg)
            stream.synchronize()
        finally:
            nv.set_lane(prev)


class LazyClips:
    """Sequence of synthetic clips generated on demand (each rank builds only
    the clips it owns): clip i = `iccad_like_clip(seed=seed0 + i)`."""

    def __init__(self, n, seed0=0, side=2048):
        self.n, self.seed0, self.side = n, seed0, side

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        from .inputs import iccad_like_clip
        if not 0 <= i < self.n:
            raise IndexError(i)
        return iccad_like_clip(seed=self.seed0 + i, n=self.side)
