"""Synthetic benchmark inputs (host side; they define workloads, they are not
on the hot path).

* `synthetic_kernel_arrays` -- the deterministic SOCS kernel generator of the
  reference (`gen_synthetic_kernels`, litho.py:213-256), bit-identical output.
* `iccad_like_clip` -- SURVEY.md Appendix B metal-layer clip generator.
* `two_bar_layout` -- the reference's AC-5 / quickstart target
  (test_acceptance.py:31).
"""

from __future__ import annotations

import numpy as np


def synthetic_kernel_arrays(side, n_k, seed=0, defocus_scale=1.25):
    """Returns ((coeffs c128 [n_k,K,K], weights f64 [n_k]) for focus, same for
    defocus).  Kernel 0 is a Gaussian; kernel i > 0 is that Gaussian times a
    plane wave of frequency pi*i/side at a seeded angle and phase; each kernel
    has unit energy; weights 0.45^i normalised so a fully lit mask peaks at 1.
    """
    if side < 3 or side % 2 == 0:
        raise ValueError(f"kernel side must be odd and >= 3, got {side}")
    if n_k < 1:
        raise ValueError(f"kernel count must be >= 1, got {n_k}")
    gen = np.random.default_rng(seed)
    half = side // 2
    gy, gx = np.mgrid[0:side, 0:side]
    dx = gx - half
    dy = gy - half
    rr = dx.astype(np.float64) ** 2 + dy.astype(np.float64) ** 2
    theta = gen.uniform(0.0, 2 * np.pi, size=n_k)   # drawn first: shared by both sets
    phi0 = gen.uniform(0.0, 2 * np.pi, size=n_k)

    def make(sigma):
        stack = np.empty((n_k, side, side), dtype=np.complex128)
        wts = np.empty(n_k)
        envelope = np.exp(-rr / (2.0 * sigma ** 2))
        for i in range(n_k):
            if i == 0:
                h = envelope.astype(np.complex128)
            else:
                kf = np.pi * i / side
                wave = kf * (np.cos(theta[i]) * dx + np.sin(theta[i]) * dy)
                h = envelope * np.exp(1j * (wave + phi0[i]))
            stack[i] = h / np.sqrt(np.sum(np.abs(h) ** 2))
            wts[i] = 0.45 ** i
        full = 0.0
        for i in range(n_k):
            full += wts[i] * abs(stack[i].sum()) ** 2
        return stack, wts / full

    s0 = side / 6.0
    return make(s0), make(s0 * defocus_scale)


def rect_layout(side, rects):
    """Pixels whose centres fall in [x, x+w) x [y, y+h) are lit."""
    g = np.zeros((side, side), dtype=np.uint8)
    for x, y, w, h in rects:
        g[y:y + h, x:x + w] = 1
    return g


def two_bar_layout():
    """parse_layout("SIZE 512\\nRECT 150 120 70 270\\nRECT 290 120 70 270\\n"):
    BASELINE configs[0] (test_acceptance.py:31)."""
    return rect_layout(512, [(150, 120, 70, 270), (290, 120, 70, 270)])


def iccad_like_clip(seed=0, n=2048, n_wires=14, lo=512, hi=1536, wmin=60, wmax=90,
                    lmin=200, lmax=800, spacing=60, tries=5000):
    """Manhattan wires placed by rejection sampling."""
    gen = np.random.default_rng(seed)
    g = np.zeros((n, n), dtype=np.uint8)
    placed = 0
    attempt = 0
    while placed < n_wires and attempt < tries:
        attempt += 1
        w = int(gen.integers(wmin, wmax + 1))
        ln = int(gen.integers(lmin, lmax + 1))
        bw, bh = (ln, w) if gen.random() < 0.5 else (w, ln)
        x = int(gen.integers(lo, hi - bw))
        y = int(gen.integers(lo, hi - bh))
        if g[max(0, y - spacing):min(n, y + bh + spacing),
             max(0, x - spacing):min(n, x + bw + spacing)].any():
            continue
        g[y:y + bh, x:x + bw] = 1
        placed += 1
    return g


def mosaic_tile(seeds, grid=(4, 4)):
    """A (4*2048)^2 periodic tile built from iccad-like clips (config 5)."""
    rows = []
    it = iter(seeds)
    for _ in range(grid[0]):
        rows.append(np.concatenate([iccad_like_clip(next(it)) for _ in range(grid[1])], axis=1))
    return np.concatenate(rows, axis=0)
