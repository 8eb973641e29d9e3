"""Grid primitives (reference fields.py).

`convolve` and `check_finite` run on the device.  `shift` and `embed_kernel`
are host-side helpers kept for API compatibility; the hot path builds its
spectra on the device (litho.KernelSet.device).
"""

from __future__ import annotations

import numpy as np

from . import _native as nv
from .errors import NumericalError

__all__ = ["shift", "embed_kernel", "convolve", "check_finite"]


def check_finite(arr, name="field"):
    """Raise NumericalError naming the first NaN/Inf pixel (fields.py:14-20)."""
    a = np.asarray(arr, dtype=np.float64)
    if a.size == 0:
        return
    dev = nv.to_dev(a.ravel())
    r = nv.reduce("nonfinite", a.size, dev)
    if r > 0:
        idx = a.size - int(r)
        y, x = np.unravel_index(idx, a.shape) if a.ndim == 2 else (0, idx)
        raise NumericalError(f"{name} is non-finite at pixel (x={x}, y={y})")


def shift(field, dx, dy, pad="zero"):
    """out(x, y) = in(x - dx, y - dy); out-of-range reads follow `pad`
    ("zero" or "replicate").  Input untouched (fields.py:23-58)."""
    src = np.asarray(field)
    h, w = src.shape
    if abs(dx) >= w or abs(dy) >= h:
        raise ValueError(f"shift ({dx}, {dy}) exceeds grid dimensions {w}x{h}")
    if pad not in ("zero", "replicate"):
        raise ValueError(f"unknown pad mode {pad!r}")
    ys = np.arange(h) - dy
    xs = np.arange(w) - dx
    inside = ((ys >= 0) & (ys < h))[:, None] & ((xs >= 0) & (xs < w))[None, :]
    out = src[np.clip(ys, 0, h - 1)][:, np.clip(xs, 0, w - 1)].copy()
    if pad == "zero":
        out[~inside] = 0
    return out


def embed_kernel(coeffs, shape):
    """K x K taps placed so the centre tap sits at (0, 0) of the grid,
    wrapping periodically (fields.py:61-74)."""
    c = np.asarray(coeffs, dtype=np.complex128)
    k = c.shape[0]
    h, w = shape
    if k > h or k > w:
        raise ValueError(f"kernel side {k} exceeds grid {w}x{h}")
    out = np.zeros(shape, dtype=np.complex128)
    out[np.ix_((np.arange(k) - k // 2) % h, (np.arange(k) - k // 2) % w)] = c
    return out


def convolve(mask, kernel):
    """Circular convolution of a real grid with one optical kernel
    (fields.py:77-87), computed by the device FFT engine."""
    from .litho import KernelSet, OpticalKernel
    coeffs = np.asarray(getattr(kernel, "coeffs", kernel), dtype=np.complex128)
    m = np.asarray(mask, dtype=np.float64)
    if coeffs.ndim != 2 or coeffs.shape[0] != coeffs.shape[1]:
        raise ValueError("kernel coefficients must be a square matrix")
    k = coeffs.shape[0]
    if k > m.shape[0] or k > m.shape[1]:
        raise ValueError(f"kernel side {k} exceeds grid {m.shape[1]}x{m.shape[0]}")
    ks = getattr(kernel, "_single_set", None)
    if ks is None:
        ks = KernelSet([OpticalKernel(coeffs, 1.0)], "focus")
        if isinstance(kernel, OpticalKernel):
            kernel._single_set = ks
    dks = ks.device(m.shape)
    out = nv.empty(m.shape, np.complex128)
    md = nv.to_dev(m)
    nv.check(nv.lib().lsopc_convolve(dks.plan.handle, dks.handle, nv.ptr(md), nv.ptr(out), nv.stream()))
    return nv.to_host(out)
