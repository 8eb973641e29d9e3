"""GPU greedy fracture / shot count (lsopc_fracture_dev)
against the reference's rectangle lists (tests/golden/fracture.npz, made by
the real reference's metrics.fracture) and against the host implementation,
which is itself pinned to the golden lists and to an exhaustive search
(test_native_abi.py).  Rectangle lists must be identical, in order."""

import os
import time

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2303_12529_b200 import metrics  # noqa: E402


def dev(m):
    return torch.as_tensor(np.ascontiguousarray(m, dtype=np.uint8), device="cuda")


def both(m):
    return metrics.fracture(dev(m)), metrics.fracture(np.asarray(m, dtype=np.uint8))


def test_device_fracture_matches_reference_rect_lists():
    g = golden("fracture")
    for i in range(12):
        ref = [tuple(int(v) for v in r) for r in g[f"rects{i}"]]
        assert metrics.fracture(dev(g[f"mask{i}"])) == ref, i
        assert metrics.shot_count(dev(g[f"mask{i}"])) == len(ref), i


def test_device_fracture_translation_and_edges():
    g = golden("fracture")
    for i in range(12):
        m = g[f"mask{i}"]
        ref = [tuple(int(v) for v in r) for r in g[f"rects{i}"]]
        for oy, ox, H, W in ((5, 9, 80, 96), (0, 0, m.shape[0] + 3, m.shape[1] + 7),
                             (7, 0, m.shape[0] + 7, m.shape[1])):
            big = np.zeros((H, W), dtype=np.uint8)
            big[oy:oy + m.shape[0], ox:ox + m.shape[1]] = m
            assert metrics.fracture(dev(big)) == [(x + ox, y + oy, w, h) for x, y, w, h in ref], (i, oy, ox)


def test_device_fracture_random_masks_match_host():
    """Random masks of many shapes and densities, including boxes up to 8192
    columns wide (256 columns per lane chunk) and single rows / columns."""
    rng = np.random.default_rng(11)
    shapes = [(1, 1), (1, 37), (41, 1), (7, 9), (33, 65), (100, 3), (64, 1000), (300, 300), (17, 8192),
              (2, 4000)]
    for H, W in shapes:
        for p in (0.3, 0.7, 0.95):
            m = (rng.random((H, W)) < p).astype(np.uint8)
            d, h = both(m)
            assert d == h, (H, W, p)


def test_device_fracture_blocky_masks_match_host():
    """Manhattan masks like optimised OPC masks (large rectangles, jogs)."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        H, W = (int(v) for v in rng.integers(50, 700, 2))
        m = np.zeros((H, W), dtype=np.uint8)
        for _ in range(int(rng.integers(3, 40))):
            h, w = (int(v) for v in rng.integers(2, 120, 2))
            y, x = int(rng.integers(0, max(1, H - h))), int(rng.integers(0, max(1, W - w)))
            m[y:y + h, x:x + w] ^= 1
        d, hh = both(m)
        assert d == hh, trial


def test_device_fracture_round_budget_continues_on_host(monkeypatch):
    """A round budget smaller than the shot count hands the remaining mask
    to the host algorithm; the list is unchanged."""
    g = golden("fracture")
    monkeypatch.setenv("LSOPC_B200_FRACTURE_ROUNDS", "7")
    for i in (1, 2, 5):
        ref = [tuple(int(v) for v in r) for r in g[f"rects{i}"]]
        assert metrics.fracture(dev(g[f"mask{i}"])) == ref, i


def test_device_fracture_box_too_large_falls_back():
    """A lit box too large for the cluster's shared memory (2048 x 2048,
    uint16 heights = 8 MB) runs the host algorithm on the device mask."""
    rng = np.random.default_rng(5)
    m = (rng.random((2048, 2048)) < 0.9).astype(np.uint8)
    m[:, :1500] = 0
    m[0, 0] = m[2047, 2047] = 1
    d, h = both(m)
    assert d == h


def test_device_shot_count_clip2048_solve():
    """configs[1]: the shot count of the 2048^2 solve's final mask (the
    reference's own: 240 shots) and the device time of the count."""
    import paper_2303_12529_b200 as b2
    g = golden("clip2048_solve")
    from oracle import lsopc_oracle as o
    clip = o.iccad_like_clip(0)
    mask = np.unpackbits(g["mask_packed"])[:clip.size].reshape(clip.shape)
    md = dev(mask)
    assert metrics.shot_count(md) == int(g["metrics"][2])
    assert metrics.fracture(md) == metrics.fracture(mask)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        metrics.shot_count(md)
    dt = (time.perf_counter() - t0) / 5
    print(f"device shot count 2048^2 final mask: {dt * 1e3:.3f} ms (240 shots)")
    r = b2.optimize(clip, *b2.gen_synthetic_kernels(35, 24, seed=4), b2.OptConfig(precision="fp32"))
    assert r.metrics.shots == metrics.shot_count(r.final_mask)
