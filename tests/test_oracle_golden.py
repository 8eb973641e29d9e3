"""Pin the numpy oracle to golden vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import lsopc_oracle as o


def kset(g, side, n_k, seed, tag):
    return g[f"{side}_{n_k}_{seed}_{tag}_c"], g[f"{side}_{n_k}_{seed}_{tag}_w"]


def test_synthetic_kernels_bit_exact():
    g = golden("kernels")
    for side, n_k, seed in [(9, 2, 0), (9, 2, 3), (17, 4, 1), (35, 8, 4), (7, 2, 0)]:
        f, d = o.synthetic_kernels(side, n_k, seed)
        for tag, (c, w) in (("f", f), ("d", d)):
            assert np.array_equal(c, g[f"{side}_{n_k}_{seed}_{tag}_c"])
            assert np.array_equal(w, g[f"{side}_{n_k}_{seed}_{tag}_w"])


def test_synthetic_kernels_35_24_hash():
    import hashlib
    g = golden("kernels")
    f, d = o.synthetic_kernels(35, 24, 4)
    for tag, (c, w) in (("f", f), ("d", d)):
        assert hashlib.sha256(c.tobytes()).digest() == g[f"35_24_4_{tag}_sha"].tobytes()
        assert np.array_equal(w, g[f"35_24_4_{tag}_w"])


def test_intensity_matches_reference():
    g = golden("forward")
    k = golden("kernels")
    f, d = kset(k, 9, 2, 3, "f"), kset(k, 9, 2, 3, "d")
    m = g["rand64_mask"]
    for key, ks, dose in (("I_nom", f, 1.0), ("I_out", f, 1.02), ("I_in", d, 0.98)):
        out = o.intensity(m, ks[0], ks[1], dose)
        ref = g[f"rand64_{key}"]
        assert np.abs(out - ref).max() <= 1e-13 * ref.max()


def test_corners_match_reference():
    g = golden("forward")
    k = golden("kernels")
    f, d = kset(k, 9, 2, 3, "f"), kset(k, 9, 2, 3, "d")
    soft = o.corners(g["bin32_mask"], f, d, binarize=False)
    hard = o.corners(g["bin32_mask"], f, d, binarize=True)
    for c, key in (("nominal", "nom"), ("inner", "in"), ("outer", "out")):
        assert np.abs(soft[c] - g[f"bin32_Z_{key}"]).max() <= 1e-13
        assert np.array_equal(hard[c], g[f"bin32_H_{key}"])


@pytest.mark.parametrize("seed", [0, 3])
def test_gradients_match_reference(seed):
    g = golden("gradients")
    k = golden("kernels")
    f, d = kset(k, 9, 2, seed, "f"), kset(k, 9, 2, seed, "d")
    target = g[f"s{seed}_target"]
    mask = target.astype(np.float64)
    p = o.corners(mask, f, d, binarize=False)
    gi = o.ilt_grad(mask, p["nominal"], target, f)
    gp = o.pvb_grad(mask, p["inner"], p["outer"], target, f, d)
    for out, ref in ((gi, g[f"s{seed}_g_ilt"]), (gp, g[f"s{seed}_g_pvb"])):
        assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    assert abs(o.ilt_loss(p["nominal"], target) - g[f"s{seed}_l_ilt"]) <= 1e-12 * g[f"s{seed}_l_ilt"]
    assert abs(o.pvb_loss(p["inner"], p["outer"], target) - g[f"s{seed}_l_pvb"]) <= 1e-12 * g[f"s{seed}_l_pvb"]


def test_geometry_and_curvature_bit_exact():
    g = golden("levelset")
    gx, gy, gxx, gyy, gxy = o.geometry(g["phi"])
    for name, arr in zip(("gx", "gy", "gxx", "gyy", "gxy"), (gx, gy, gxx, gyy, gxy)):
        assert np.array_equal(arr, g[name]), name
    assert np.array_equal(np.hypot(gx, gy), g["mag"])
    assert np.array_equal(o.kappa(g["phi"], g["mod"], 0.9), g["kappa"])


def test_tsdf_bit_exact():
    g = golden("levelset")
    for i in range(4):
        assert np.array_equal(o.tsdf(g[f"tsdf_mask{i}"]), g[f"tsdf_phi{i}"])
    t = o.rect_layout(128, [(25, 30, 30, 50), (70, 60, 40, 40)])
    assert np.array_equal(o.tsdf(t, 20.0, -7.0), g["tsdf_two_rect"])


@pytest.mark.parametrize("tag", ["on", "off"])
def test_optimize_rect128_trajectory(tag):
    g = golden("optimize")
    k = golden("kernels")
    f, d = kset(k, 17, 4, 1, "f"), kset(k, 17, 4, 1, "d")
    t = o.rect_layout(128, [(25, 30, 30, 50), (70, 60, 40, 40)])
    cfg = o.Cfg(max_iters=15, use_curvature=(tag == "on"))
    r = o.optimize(t, f, d, cfg)
    hist = np.array(r.history)
    ref = g[f"rect128_{tag}_hist"]
    assert hist.shape == ref.shape
    assert np.allclose(hist, ref, rtol=1e-9, atol=1e-12)
    assert np.array_equal(r.final_mask, g[f"rect128_{tag}_mask"])
    assert np.abs(r.best_phi - g[f"rect128_{tag}_phi"]).max() <= 1e-9
    l2, pvb, _shots, iters = g[f"rect128_{tag}_metrics"]
    assert (r.l2, r.pvband, len(r.history)) == (l2, pvb, iters)


def test_two_bar_layout_and_clip_generator():
    t = o.two_bar_512()
    assert t.sum() == 2 * 70 * 270
    assert [int(o.iccad_like_clip(s).sum()) for s in (0, 1, 2)] == [333562, 308514, 334395]


def test_modulation_search_matches_reference():
    """optimizer.py:294-341 restated; fixture from the real reference (make_golden.py)."""
    g = golden("modsearch")
    f, d = o.synthetic_kernels(9, 2, 2)
    t = g["target"]
    phi = o.tsdf(t)
    r = o.modulation_search(phi, t, f, d, None, num_samples=5, eval_steps=3)
    assert np.array_equal(np.array(r["candidates"]), g["default_candidates"])
    assert r["best_delta_h"] == float(g["default_best"])
    r = o.modulation_search(phi, t, f, d, o.Cfg(curvature_weight=0.0), num_samples=5, eval_steps=3)
    assert np.array_equal(np.array(r["candidates"]), g["nocurvw_candidates"])
    assert r["best_delta_h"] == float(g["nocurvw_best"])


def test_oracle_spectra_match_reference_stacked_ffts():
    """`o.spectra` / `o.reverse_freq` against the reference's own
    KernelSet.stacked_ffts (litho.py:71-82), tests/golden/make_spectra.py."""
    g = golden("spectra")
    for side, n_k, seed, shape in [(9, 2, 3, (32, 64)), (17, 4, 1, (64, 64)), (7, 2, 0, (16, 128))]:
        f, d = o.synthetic_kernels(side, n_k, seed)
        for tag, (c, w) in (("f", f), ("d", d)):
            key = f"{side}_{n_k}_{seed}_{tag}_{shape[0]}x{shape[1]}"
            hf = o.spectra(c, shape)
            assert np.abs(hf - g[key + "_hf"]).max() <= 1e-12 * np.abs(g[key + "_hf"]).max()
            assert np.abs(o.reverse_freq(hf) - g[key + "_hrot"]).max() <= 1e-12 * np.abs(g[key + "_hf"]).max()
            assert np.array_equal(w, g[key + "_sigma"])
