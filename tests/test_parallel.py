"""Clip-parallel (multi-GPU) host logic, exercised with world_size-2 gloo
process groups on CPU (the device solver is replaced by a stub)."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_12529_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stub_solver(target, f, d, cfg):
    m = SimpleNamespace(l2=int(target.sum()), pvband=int(target[0].sum()), shots=int(target.shape[0]))
    return SimpleNamespace(metrics=m, iters_run=int(target.sum()) % 7, wall_time=0.0)


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        targets = [np.full((4, 4), i % 3, dtype=np.uint8) * (i + 1) for i in range(n)]
        recs, secs = parallel.optimize_batch(targets, None, None, None, solver=_stub_solver)
        mx = parallel.max_over_ranks(float(rank + 1))
        q.put((rank, [(r.index, r.rank, r.l2, r.pvband, r.shots, r.iters) for r in recs], secs, mx))
    finally:
        dist.destroy_process_group()


def test_shard_round_robin_covers_disjointly():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard(n, r, world) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            for r, p in enumerate(parts):
                assert all(i % world == r for i in p)
    with pytest.raises(ValueError):
        parallel.shard(4, 2, 2)


def test_single_process_batch_without_group():
    targets = [np.eye(3, dtype=np.uint8) * i for i in range(5)]
    recs, secs = parallel.optimize_batch(targets, None, None, None, solver=_stub_solver)
    assert [r.index for r in recs] == list(range(5))
    assert all(r.rank == 0 for r in recs) and secs >= 0.0
    assert parallel.max_over_ranks(3.5) == 3.5


def test_world2_gloo_batch_gathers_all_clips_in_order():
    world, n = 2, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    expect = []
    for i in range(n):
        t = np.full((4, 4), i % 3, dtype=np.uint8) * (i + 1)
        s = _stub_solver(t, None, None, None)
        expect.append((i, i % world, s.metrics.l2, s.metrics.pvband, s.metrics.shots, s.iters_run))
    for rank, recs, secs, mx in out:
        assert recs == expect          # every rank sees all clips, ordered, with the owner rank
        assert mx == float(world)      # max over ranks of rank + 1
        assert secs >= 0.0


def test_lazy_clips_are_deterministic():
    c = parallel.LazyClips(3, seed0=0, side=2048)
    assert len(c) == 3
    a = c[0]
    assert a.shape == (2048, 2048) and a.dtype == np.uint8
    assert np.array_equal(a, c[0])
    with pytest.raises(IndexError):
        c[3]


# ---- modulation_search candidates sharded over ranks ----------

def _stub_score(dh):
    # ties at dh = +-5 (loss 0): the reference's tie-break picks -5.0
    return abs(abs(dh) - 5.0)


def _ms_target():
    t = np.zeros((8, 8), dtype=np.uint8)
    t[2:6, 3:7] = 1
    return t


def _ms_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        phi = SimpleNamespace(phi=np.linspace(-3, 3, 64).reshape(8, 8))
        cfg = SimpleNamespace(__dict__={})
        from paper_2303_12529_b200 import OptConfig
        r, secs = parallel.modulation_search_sharded(phi, _ms_target(), None, None, OptConfig(), num_samples=41,
                                                     scorer=_stub_score)
        q.put((rank, r.best_delta_h, r.candidates, r.m_gt.tolist(), secs))
    finally:
        dist.destroy_process_group()


def test_modulation_search_sharded_single_process():
    from paper_2303_12529_b200 import OptConfig
    phi = SimpleNamespace(phi=np.linspace(-3, 3, 64).reshape(8, 8))
    r, secs = parallel.modulation_search_sharded(phi, _ms_target(), None, None, OptConfig(), num_samples=41,
                                                 scorer=_stub_score)
    offsets = list(np.linspace(-20.0, 20.0, 41))
    assert [dh for dh, _ in r.candidates] == offsets
    assert [l for _, l in r.candidates] == [_stub_score(dh) for dh in offsets]
    assert r.best_delta_h == -5.0
    assert np.array_equal(r.m_gt, (phi.phi - 5.0 >= 0).astype(np.float64))
    r1, _ = parallel.modulation_search_sharded(phi, _ms_target(), None, None, OptConfig(), num_samples=1,
                                               scorer=_stub_score)
    assert r1.best_delta_h == 0.0 and r1.candidates == [(0.0, 5.0)]


def test_world2_gloo_modulation_search_agrees_on_every_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ms_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    offsets = list(np.linspace(-20.0, 20.0, 41))
    for rank, best, cands, m_gt, secs in out:
        assert best == -5.0
        assert [dh for dh, _ in cands] == offsets
        assert [l for _, l in cands] == [_stub_score(dh) for dh in offsets]
        assert secs >= 0.0
    assert out[0][3] == out[1][3]
