"""Tall / wide geometries against the oracle.

8192-point columns (8192 x 256) take the split plan (Grid::vsplit): the
direct K0 spectra build, the radix-4 plane combine inside the row passes and
2048-point column passes on the virtual 2048 x 4W grid -- in both tiers.
8192-point rows (256 x 8192) take the tall-row TMA row passes (fp32).
4096-point sides (the fp64 tier's largest single-plan sides) are checked too.
Everything is checked against the numpy oracle on the same inputs with the
production kernel model (24 + 24 kernels, K = 35, seed 4):

                             fp32                 fp64
  intensity (3 corners)      rel-to-max 1e-5      1e-10   (litho.py:114-126)
  soft prints                abs 1e-5             1e-10   (litho.py:141-154)
  ILT / PVB gradients        rel-to-max 2e-5      1e-9    (optimizer.py:99-129)
  6-iteration optimize       history rtol 1e-4    1e-8    (optimizer.py:204-284)

The oracle runs on the host's cores through scipy.fft (same pocketfft as
numpy).  The pre-split fp32 path (4-CTA cluster columns, four-step F1) is
compared with the split plan in test_tiled.py.
"""

import os

import numpy as np
import pytest

from oracle import lsopc_oracle as o

pytestmark = pytest.mark.gpu

b2 = pytest.importorskip("paper_2303_12529_b200")
from paper_2303_12529_b200 import _native as nv  # noqa: E402

CASES = [("fp32", (8192, 256)), ("fp32", (256, 8192)), ("fp64", (8192, 256)),
         # 4096-point sides: complex128 single-column passes / one-row items, complex64 half-width items
         ("fp64", (4096, 256)), ("fp64", (256, 4096)), ("fp32", (4096, 256))]
TOL = {"fp32": dict(i=1e-5, p=1e-5, g=2e-5, h=1e-4, v=1e-3),
       "fp64": dict(i=1e-10, p=1e-10, g=1e-9, h=1e-8, v=1e-8)}


def strip_layout(shape, seed, n=40):
    """Random Manhattan rectangles 30-120 px on a tall or wide strip."""
    rng = np.random.default_rng(seed)
    t = np.zeros(shape, np.uint8)
    H, W = shape
    for _ in range(n):
        h, w = rng.integers(30, 120, size=2)
        y, x = rng.integers(0, H - h), rng.integers(0, W - w)
        t[y:y + h, x:x + w] = 1
    return t


@pytest.fixture(scope="module")
def model():
    f, d = o.synthetic_kernels(35, 24, 4)
    F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*f)], "focus")
    D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*d)], "defocus")
    return f, d, F, D


@pytest.fixture(autouse=True)
def threads():
    old = nv.get_precision()
    o.use_threads(os.cpu_count() or 1)
    yield
    o.use_threads(None)
    nv.set_precision(old)


# the oracle's results depend only on the shape (seeded target, same kernels):
# cached so the fp32 and fp64 cases of one shape share one CPU run
_ORACLE = {}


def _oracle_forward(f, d, shape):
    key = ("fwd", shape)
    if key not in _ORACLE:
        t = strip_layout(shape, sum(shape))
        m = t.astype(np.float64)
        hf_f, hf_d = o.spectra(f[0], shape), o.spectra(d[0], shape)
        ints = [o.intensity(m, arrs[0], arrs[1], dose, hf)
                for arrs, dose, hf in ((f, 1.0, hf_f), (f, 1.02, hf_f), (d, 0.98, hf_d))]
        pr = o.corners(m, f, d, binarize=False, hf_focus=hf_f, hf_defocus=hf_d)
        gi = o.ilt_grad(m, pr["nominal"], t, f, hf=hf_f)
        gp = o.pvb_grad(m, pr["inner"], pr["outer"], t, f, d, hf_focus=hf_f, hf_defocus=hf_d)
        _ORACLE[key] = (t, m, ints, pr, gi, gp)
    return _ORACLE[key]


def _oracle_history(f, d, shape):
    key = ("hist", shape)
    if key not in _ORACLE:
        t = strip_layout(shape, 7 + sum(shape))
        _ORACLE[key] = (t, np.array(o.optimize(t, f, d, o.Cfg(max_iters=6, stop_patience=10**9)).history))
    return _ORACLE[key]


def relmax(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(b).max()


@pytest.mark.parametrize("prec,shape", CASES)
def test_tall_forward_and_gradients_vs_oracle(model, prec, shape):
    f, d, F, D = model
    nv.set_precision(prec)
    tol = TOL[prec]
    t, m, ints, pr, gi_ref, gp_ref = _oracle_forward(f, d, shape)
    for ks, cond, ref in ((F, b2.NOMINAL, ints[0]), (F, b2.OUTER, ints[1]), (D, b2.INNER, ints[2])):
        out = b2.aerial_intensity(m, ks, cond)
        assert relmax(out, ref) <= tol["i"], (shape, cond.label)
    cfg = b2.OptConfig()
    p = b2.print_corners(m, F, D, cfg, binarize=False)
    for c in ("nominal", "inner", "outer"):
        assert np.abs(getattr(p, c) - pr[c]).max() <= tol["p"], (shape, c)
    gi = b2.ilt_gradient(m, pr["nominal"], t, F, cfg)
    gp = b2.pvb_gradient(m, pr["inner"], pr["outer"], t, F, D, cfg)
    assert relmax(gi, gi_ref) <= tol["g"], shape
    assert relmax(gp, gp_ref) <= tol["g"], shape


@pytest.mark.parametrize("prec,shape", CASES)
def test_tall_optimize_history_vs_oracle(model, prec, shape):
    f, d, F, D = model
    tol = TOL[prec]
    t, hr = _oracle_history(f, d, shape)
    r = b2.optimize(t, F, D, b2.OptConfig(max_iters=6, stop_patience=10**9, precision=prec))
    h = np.array([[x.l_ilt, x.l_pvb, x.l_dso, x.dt, x.max_v, x.max_step, x.max_grad_mag]
                  for x in r.loss_history])
    assert h.shape == hr.shape == (6, 7)
    assert np.allclose(h[:, :3], hr[:, :3], rtol=tol["h"]), (shape, h[:, :3], hr[:, :3])
    # dt / max|v| are maxima over the whole grid (curvature-dominated pixels)
    assert np.allclose(h[:, 3:5], hr[:, 3:5], rtol=tol["v"]), (shape, h[:, 3:5], hr[:, 3:5])


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_split_plan_spectra_vs_oracle(model, prec):
    """K0 of a split plan (8192 rows: direct separable DFT, plane-ordered
    storage) downloaded through stacked_ffts against the oracle's
    embed + FFT2 (litho.py:71-82, fields.py:61-74)."""
    f, d, F, D = model
    nv.set_precision(prec)
    shape = (8192, 256)
    hf, hrot, sigma = F.stacked_ffts(shape)
    ref = o.spectra(f[0], shape)
    tol = 1e-12 if prec == "fp64" else 2e-7
    assert np.abs(hf - ref).max() <= tol * np.abs(ref).max(), prec
    assert np.array_equal(sigma, np.asarray(f[1], np.float64))


@pytest.mark.parametrize("prec,shape", [("fp64", (8192, 512)), ("fp64", (8192, 1024)), ("fp32", (8192, 2048)),
                                        ("fp32", (8192, 1024))])
def test_split_plan_widths_vs_oracle(prec, shape):
    """Every split-plan item geometry (Q = 4W'/W rows per plane: fp64 W = 512
    -> Q = 2, W = 1024 -> Q = 1; fp32 W = 1024 -> Q = 2, W = 2048 -> Q = 1)
    against the oracle, with a small kernel set (4 + 4 kernels, K = 17) to
    keep the CPU side short: intensity at the three corners and the ILT
    gradient."""
    nv.set_precision(prec)
    tol = TOL[prec]
    f, d = o.synthetic_kernels(17, 4, 2)
    F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*f)], "focus")
    D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*d)], "defocus")
    t = strip_layout(shape, 3 + sum(shape), n=60)
    m = t.astype(np.float64)
    hf_f, hf_d = o.spectra(f[0], shape), o.spectra(d[0], shape)
    for arrs, ks, cond, hf in ((f, F, b2.NOMINAL, hf_f), (f, F, b2.OUTER, hf_f), (d, D, b2.INNER, hf_d)):
        assert relmax(b2.aerial_intensity(m, ks, cond), o.intensity(m, arrs[0], arrs[1], cond.dose, hf)) <= tol["i"]
    z = o.corners(m, f, d, binarize=False, hf_focus=hf_f, hf_defocus=hf_d)["nominal"]
    gi = b2.ilt_gradient(m, z, t, F, b2.OptConfig())
    assert relmax(gi, o.ilt_grad(m, z, t, f, hf=hf_f)) <= tol["g"], shape


def test_fp64_plan_limits():
    """The fp64 tier takes 8192 x W grids for 256 <= W <= 1024 (split plan)
    and rejects wider 8192-row grids and 8192-point rows with ValueError
    (the plan's message names the limit)."""
    nv.set_precision("fp64")
    f, d = o.synthetic_kernels(7, 1, 0)
    F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*f)], "focus")
    for shape in ((8192, 2048), (256, 8192)):
        with pytest.raises(ValueError, match="FP64 tier"):
            b2.aerial_intensity(np.zeros(shape), F)
    out = b2.aerial_intensity(np.zeros((8192, 512)), F)
    assert out.shape == (8192, 512) and not out.any()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_split_plan_convolve_vs_numpy(prec):
    """fields.convolve (fields.py:77-87) on a split plan (8192 x 256): the
    field A_0 comes out of the split F2 in natural row order."""
    nv.set_precision(prec)
    f, _ = o.synthetic_kernels(11, 1, 5)
    k = f[0][0]
    t = strip_layout((8192, 256), 99, n=30).astype(np.float64)
    out = b2.convolve(t, b2.OpticalKernel(k, 1.0))
    ref = np.fft.ifft2(np.fft.fft2(t) * np.fft.fft2(o.embed(k, t.shape)))
    tol = 1e-12 if prec == "fp64" else 2e-6
    assert np.abs(out - ref).max() <= tol * np.abs(ref).max(), prec
