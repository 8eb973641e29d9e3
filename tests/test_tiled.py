"""Oversized-tile strip decomposition (BASELINE configs[4]): host logic with
world_size 2/4 gloo groups on CPU, and device parity against the single-tile
optimize on the GPU (ranks sharing one GPU over gloo)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_12529_b200 import tiled


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args, timeout=300):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=timeout) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_strip_geometry():
    for W, world, K in [(1024, 4, 35), (8192, 8, 35), (2048, 2, 17), (512, 1, 35)]:
        strips = [tiled.strip_geometry(256, W, world, r, K) for r in range(world)]
        covered = np.concatenate([np.arange(s.x0, s.x1) for s in strips])
        assert np.array_equal(np.sort(covered), np.arange(W))
        for s in strips:
            i0, i1 = s.interior
            assert s.ww & (s.ww - 1) == 0 and s.ww <= W
            assert i0 >= min(s.halo, i0) and (world == 1 or (i0 >= s.halo and s.ww - i1 >= s.halo))
            assert np.array_equal(s.columns()[i0:i1], np.arange(s.x0, s.x1))
    s = tiled.strip_geometry(8192, 8192, 8, 3, 35)
    assert (s.ww, s.hl, s.interior) == (2048, 512, (512, 1536))
    assert tiled.strip_geometry(64, 1024, 4, 0, 35).stencil_bounds() == (128, 512)
    assert tiled.strip_geometry(64, 1024, 4, 3, 35).stencil_bounds() == (0, 384)
    with pytest.raises(ValueError):
        tiled.strip_geometry(64, 100, 3, 0, 35)
    with pytest.raises(ValueError):
        tiled.strip_geometry(64, 128, 2, 0, 35)
    # row strips: the same geometry in the transposed frame
    r = tiled.strip_geometry(8192, 8192, 8, 3, 35, axis=0)
    assert (r.ww, r.hl, r.interior, r.window_shape) == (2048, 512, (512, 1536), (2048, 8192))
    assert tiled.strip_geometry(1024, 64, 4, 0, 35, axis=0).stencil_bounds() == (128, 512)


def test_strip_layout_and_auto_strips():
    """Several strips per rank: unequal interiors (floor(i L / n)) with one
    common window; the automatic count minimises the window area per rank
    among windows of 512..2048 lines (fp32) or a legal fp64 plan (8192 x
    <=1024, column strips)."""
    for L, n, K in [(8192, 5, 35), (8192, 9, 35), (1024, 3, 35), (1000, 7, 17)]:
        strips = tiled.strip_layout(64, L, n, K)
        assert len({s.ww for s in strips}) == 1
        covered = np.concatenate([np.arange(s.x0, s.x1) for s in strips])
        assert np.array_equal(covered, np.arange(L))
        for s in strips:
            i0, i1 = s.interior
            assert i0 >= s.halo and s.ww - i1 >= s.halo
            assert np.array_equal(s.columns()[i0:i1], np.arange(s.x0, s.x1))
    assert [s.ww for s in tiled.strip_layout(64, 8192, 5, 35)][0] == 2048
    assert tiled.auto_strips(8192, 8192, 1, 35, 0, "fp32") == 9   # 9 x 1024-line windows
    assert tiled.auto_strips(8192, 8192, 8, 35, 0, "fp32") == 3   # 3 x 512 per rank
    assert tiled.auto_strips(8192, 8192, 2, 35, 0, "fp32") == 5
    assert tiled.auto_strips(8192, 8192, 1, 35, 1, "fp64") == 9   # 8192 x 1024, split plan
    assert tiled.auto_strips(256, 1024, 1, 35, 1, "fp64") == 1
    assert tiled.auto_strips(256, 1024, 2, 35, 1, "fp32") == 1
    with pytest.raises(ValueError):
        tiled.auto_strips(8192, 8192, 1, 35, 0, "fp64")  # complex128 rows stop at 4096 points


def test_local_halo_exchange():
    """Strips held by one process refresh each other's halos (ring)."""
    for axis in (1, 0):
        strips = tiled.strip_layout(8, 1000, 5, 17, 1) if axis == 1 else tiled.strip_layout(1000, 8, 5, 17, 0)
        phis = []
        for s in strips:
            p = torch.full((8, s.ww), -1.0, dtype=torch.float64)
            i0, i1 = s.interior
            p[:, i0:i1] = torch.as_tensor(s.columns()[i0:i1], dtype=torch.float64)
            phis.append(p.t().contiguous() if axis == 0 else p)
        tiled.exchange_local_halos(phis, strips, wrap=True)
        for s, p in zip(strips, phis):
            p = p.t() if axis == 0 else p
            i0, i1 = s.interior
            h = s.halo
            assert np.array_equal(p[:, i0 - h:i1 + h].numpy(),
                                  np.broadcast_to(s.columns()[i0 - h:i1 + h], (8, i1 - i0 + 2 * h)))


def _multi_halo_worker(rank, world, port, q, W, K, m):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = tiled.strip_layout(8, W, world * m, K)[rank * m:(rank + 1) * m]
        phis = []
        for s in mine:
            p = torch.full((8, s.ww), -1.0, dtype=torch.float64)
            i0, i1 = s.interior
            p[:, i0:i1] = torch.as_tensor(s.columns()[i0:i1], dtype=torch.float64)
            phis.append(p)
        tiled.exchange_local_halos(phis, mine, wrap=False)
        tiled.exchange_halos(phis[0], mine[0], tags=False, last=(phis[-1], mine[-1]))
        q.put((rank, [p.numpy() for p in phis], [(s.columns(), s.interior, s.halo) for s in mine]))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_several_strips_per_rank_gloo():
    """Two ranks x three strips: device-local copies inside a rank, positional
    P2P (no tags) between the ranks' edge strips, wrapping."""
    for rank, phis, geo in _run(2, _multi_halo_worker, 1200, 17, 3):
        for p, (cols, (i0, i1), h) in zip(phis, geo):
            assert np.array_equal(p[:, i0 - h:i1 + h], np.broadcast_to(cols[i0 - h:i1 + h], (8, i1 - i0 + 2 * h)))


def _gather_worker(rank, world, port, q, axis):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 5 + 2 * rank  # interiors of different extent per rank
        t = torch.arange(3 * n, dtype=torch.float64).reshape((3, n) if axis == 1 else (n, 3)) + 100 * rank
        q.put((rank, [x.numpy() for x in tiled._all_gather_var(t, axis)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("axis", [0, 1])
def test_all_gather_of_unequal_interiors(axis):
    """The NCCL assembly path pads each rank's interior block to the widest
    and trims it back (strip interiors differ by a line when n does not
    divide the tile)."""
    for rank, parts in _run(2, _gather_worker, axis):
        for r, x in enumerate(parts):
            n = 5 + 2 * r
            ref = np.arange(3 * n, dtype=np.float64).reshape((3, n) if axis == 1 else (n, 3)) + 100 * r
            assert np.array_equal(x, ref)


def _halo_worker(rank, world, port, q, W, K, tags, axis=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = tiled.strip_geometry(8, W, world, rank, K) if axis == 1 else tiled.strip_geometry(W, 8, world, rank, K, 0)
        phi = torch.full((8, s.ww), -1.0, dtype=torch.float64)
        i0, i1 = s.interior
        phi[:, i0:i1] = torch.as_tensor(s.columns()[i0:i1], dtype=torch.float64)
        if axis == 0:  # row strips: the window is (ww x 8), lines are rows
            phi = phi.t().contiguous()
        tiled.exchange_halos(phi, s, tags=tags)
        if axis == 0:
            phi = phi.t().contiguous()
        q.put((rank, phi.numpy(), s.columns(), s.interior, s.halo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("axis", [1, 0])
@pytest.mark.parametrize("tags", [True, False])
@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_gloo(world, tags, axis):
    """tags=False: every message carries the same tag, so the two messages
    between the ranks of a world-2 ring are matched by position only -- the
    way NCCL matches them (it ignores P2P tags).  axis 0: row strips."""
    W, K = 1024, 35
    for rank, phi, cols, (i0, i1), h in _run(world, _halo_worker, W, K, tags, axis):
        # interior and HALO columns on each side hold the global column index (wrapping)
        assert np.array_equal(phi[:, i0 - h:i1 + h], np.broadcast_to(cols[i0 - h:i1 + h], (8, i1 - i0 + 2 * h)))


# ---------------------------------------------------------------------------
# device parity (GPU box)

def _case():
    from conftest import golden
    kg = golden("kernels")
    t = np.zeros((256, 1024), dtype=np.uint8)
    t[60:200, 200:300] = 1    # crosses the 256-column strip boundaries
    t[100:140, 480:560] = 1
    t[30:90, 700:1000] = 1
    return t, (kg["35_8_4_f_c"], kg["35_8_4_f_w"]), (kg["35_8_4_d_c"], kg["35_8_4_d_w"])


def _ks(arrs, cond):
    import paper_2303_12529_b200 as b2
    return b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*arrs)], cond)


def _tiled_worker(rank, world, port, q, max_iters, axis=0, spr=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    torch.cuda.set_device(0)
    nv.set_precision("fp64")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, f, d = _case()
        r = tiled.optimize_tiled(t, _ks(f, "focus"), _ks(d, "defocus"), b2.OptConfig(max_iters=max_iters), axis=axis,
                                 strips_per_rank=spr)
        h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
        q.put((rank, h, r.final_mask, r.metrics.l2, r.metrics.pvband))
    finally:
        dist.destroy_process_group()


def _reference(max_iters):
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    nv.set_precision("fp64")
    t, f, d = _case()
    r = b2.optimize(t, _ks(f, "focus"), _ks(d, "defocus"), b2.OptConfig(max_iters=max_iters))
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
    return h, r.final_mask, r.metrics.l2, r.metrics.pvband


@pytest.mark.gpu
@pytest.mark.parametrize("axis", [0, 1])
def test_single_strip_is_bit_identical_to_optimize(axis):
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    nv.set_precision("fp64")
    t, f, d = _case()
    r = tiled.optimize_tiled(t, _ks(f, "focus"), _ks(d, "defocus"), b2.OptConfig(max_iters=12), axis=axis)
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
    hr, mr, l2, pvb = _reference(12)
    assert np.array_equal(h, hr)
    assert np.array_equal(r.final_mask, mr) and (r.metrics.l2, r.metrics.pvband) == (l2, pvb)


@pytest.mark.gpu
def test_two_ranks_two_strips_each_match_single_tile():
    """2 ranks x 2 strips (local copies inside a rank, P2P between ranks) on
    column strips of the 256 x 1024 case."""
    hr, mr, l2, pvb = _reference(12)
    for rank, h, mask, l2r, pvbr in _run(2, _tiled_worker, 12, 1, 2, timeout=600):
        assert np.allclose(h, hr, rtol=1e-9, atol=1e-12)
        assert np.array_equal(mask, mr)
        assert (l2r, pvbr) == (l2, pvb)


@pytest.mark.gpu
@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("world", [2, 4])
def test_strips_match_single_tile(world, axis):
    """Ranks share cuda:0 over gloo; interior results equal the full-tile run
    up to summation order of the global reductions; row (axis 0) and column
    (axis 1) strips."""
    hr, mr, l2, pvb = _reference(12)
    for rank, h, mask, l2r, pvbr in _run(world, _tiled_worker, 12, axis, timeout=600):
        assert h.shape == hr.shape
        assert np.allclose(h, hr, rtol=1e-9, atol=1e-12)
        assert np.array_equal(mask, mr)
        assert (l2r, pvbr) == (l2, pvb)


@pytest.mark.gpu
@pytest.mark.parametrize("axis", [0, 1])
def test_several_strips_in_one_process_match_single_tile(axis):
    """One process runs the tile as three strips (shared plan, phases 0/5 per
    strip, then the stop rule): the same history up to summation order, the
    same final mask and L2 / PVB as the single-tile optimize."""
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    nv.set_precision("fp64")
    t, f, d = _case()
    if axis == 0:
        t = np.ascontiguousarray(t.T)
    F, D = _ks(f, "focus"), _ks(d, "defocus")
    r = tiled.optimize_tiled(t, F, D, b2.OptConfig(max_iters=12), axis=axis, strips_per_rank=3)
    assert r.strips == 3 and r.window == ((256, 512) if axis == 1 else (512, 256))
    rr = b2.optimize(t, F, D, b2.OptConfig(max_iters=12))
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
    hr = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in rr.loss_history])
    assert h.shape == hr.shape
    assert np.allclose(h, hr, rtol=1e-9, atol=1e-12)
    assert np.array_equal(r.final_mask, rr.final_mask)
    assert (r.metrics.l2, r.metrics.pvband) == (rr.metrics.l2, rr.metrics.pvband)


@pytest.mark.gpu
def test_several_strips_with_host_phi0():
    """phi0 given on the host (windowed per strip) equals the default device
    TSDF start when phi0 is that TSDF: bit-identical histories and masks."""
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    nv.set_precision("fp64")
    t, f, d = _case()
    F, D = _ks(f, "focus"), _ks(d, "defocus")
    cfg = b2.OptConfig(max_iters=5)
    phi0 = b2.tsdf_from_mask(t, cfg.d_upper, cfg.d_lower)
    a = tiled.optimize_tiled(t, F, D, cfg, axis=1, strips_per_rank=3)
    b = tiled.optimize_tiled(t, F, D, cfg, phi0=phi0, axis=1, strips_per_rank=3)
    assert [h.l_dso for h in a.loss_history] == [h.l_dso for h in b.loss_history]
    assert np.array_equal(a.final_mask, b.final_mask) and np.array_equal(a.final_phi.phi, b.final_phi.phi)


@pytest.mark.gpu
def test_fp64_column_strips_through_split_plan_match_single_grid():
    """The fp64 configs[4] path in miniature: an 8192 x 1024 tile as three
    8192 x 512 column windows (split plan, complex128) against the same tile
    solved as one 8192 x 1024 split-plan grid (itself pinned to the oracle
    at 8192 x 256, test_tall_parity.py): history rtol 1e-9, same mask."""
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv, inputs
    nv.set_precision("fp64")
    t = np.ascontiguousarray(inputs.mosaic_tile(range(16), grid=(4, 4))[:, 2048:3072])
    fa, da = inputs.synthetic_kernel_arrays(35, 24, 4)
    F, D = _ks(fa, "focus"), _ks(da, "defocus")
    cfg = b2.OptConfig(max_iters=6, stop_patience=10**9)
    r = tiled.optimize_tiled(t, F, D, cfg, axis=1, strips_per_rank=3)
    assert r.strips == 3 and r.window == (8192, 512)
    rr = b2.optimize(t, F, D, cfg)
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
    hr = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in rr.loss_history])
    assert np.allclose(h, hr, rtol=1e-9, atol=1e-12)
    assert np.array_equal(r.final_mask, rr.final_mask)
    assert (r.metrics.l2, r.metrics.pvband) == (rr.metrics.l2, rr.metrics.pvband)


@pytest.mark.gpu
def test_configs4_tile_strips_match_full_grid_8192():
    """configs[4] at full size (parity against the single-GPU
    full-grid 8192^2 run): the 8192^2 mosaic as nine 1024 x 8192 strips in
    one process against the same tile optimised as one 8192^2 grid, fp32
    tier, 4 iterations.  The two runs use different transform lengths along
    y, so they agree to float32 rounding: losses rtol 1e-4, maxima 1e-3,
    and final masks within a handful of threshold pixels."""
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import inputs
    tile = inputs.mosaic_tile(range(16), grid=(4, 4))
    focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
    cfg = b2.OptConfig(max_iters=4, stop_patience=10**9, precision="fp32")
    r = tiled.optimize_tiled(tile, focus, defocus, cfg)
    assert r.strips == 9 and r.window == (1024, 8192)
    rr = b2.optimize(tile, focus, defocus, cfg)
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in r.loss_history])
    hr = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag] for x in rr.loss_history])
    assert h.shape == hr.shape == (4, 7)
    assert np.allclose(h[:, :3], hr[:, :3], rtol=1e-4), (h[:, :3], hr[:, :3])
    assert np.allclose(h[:, 3:], hr[:, 3:], rtol=1e-3), (h[:, 3:], hr[:, 3:])
    flips = int((r.final_mask != rr.final_mask).sum())
    assert flips <= 64, flips
    assert abs(r.metrics.l2 - rr.metrics.l2) <= 64 and abs(r.metrics.pvband - rr.metrics.pvband) <= 64


@pytest.mark.gpu
def test_tall_grid_cluster_column_passes_match_single_column_path():
    """8192-point columns (configs[4] windows): the split plan (default; 2048-
    point virtual-grid column passes), and with it disabled the 4-CTA cluster
    passes (k_pass_cluster, with and without the four-step F1 k_f1_split),
    each against the single-column cp.async passes.  Inputs bit-identical,
    outputs within float32 rounding."""
    import subprocess
    import sys
    from pathlib import Path
    script = Path(__file__).resolve().parents[1] / "scripts" / "cluster_check.py"
    # 8192 x 2048: the split plan with one row per plane in an item (Q = 1); float32 rounding of the two
    # paths' different transform orders shows at 7e-6 there (the cluster path differs by the same amount)
    legs = [("256", [], 1e-6), ("256", ["LSOPC_B200_NO_VSPLIT=1"], 1e-6),
            ("256", ["LSOPC_B200_NO_VSPLIT=1,LSOPC_B200_NO_SPLIT=1"], 1e-6), ("2048", [], 2e-5)]
    for width, extra, tol in legs:
        p = subprocess.run([sys.executable, str(script), "8192", width, *extra], capture_output=True, text=True,
                           timeout=600)
        assert p.returncode == 0, p.stdout + p.stderr
        line = p.stdout.strip().splitlines()[-1]
        rel = float(line.split("rel diff ")[1].split(",")[0])
        assert rel <= tol, (extra, line)
        assert line.endswith("final mask xor 0"), (extra, line)
