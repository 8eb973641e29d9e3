"""Mask metrics: drop-in for the reference `lsopc.metrics` (metrics.py:1-108).

L2 / PVBand are device popcounts; the greedy fracturing shot count runs on
the GPU for device masks (lsopc_fracture_dev: one thread-block cluster) and
as native host code for host masks (lsopc_fracture).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nv

__all__ = ["MetricsReport", "l2_error", "pvband", "fracture", "shot_count", "EPEReport", "epe"]


@dataclass
class MetricsReport:
    l2: int
    pvband: int
    shots: int
    wall_time: float = 0.0
    iters: int = 0

    def as_dict(self):
        return {"l2": int(self.l2), "pvband": int(self.pvband), "shots": int(self.shots),
                "wall_time_s": float(self.wall_time), "iters": int(self.iters)}


def _count_neq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0
    return int(nv.reduce("countneq", a.size, nv.to_dev(a.ravel()), nv.to_dev(b.ravel())))


def l2_error(z, z_t, pitch=1):
    """Disagreeing pixels times pitch^2 (metrics.py:39-44)."""
    return _count_neq(z, z_t) * pitch * pitch


def pvband(z_in, z_out, pitch=1):
    """XOR area of the inner and outer prints times pitch^2 (metrics.py:47-52)."""
    return _count_neq(z_in, z_out) * pitch * pitch


def _is_device(mask):
    return hasattr(mask, "is_cuda") and mask.is_cuda


def _device_u8(mask):
    t = nv.torch()
    if mask.dim() != 2:
        raise ValueError("mask must be 2-D")
    if mask.dtype != t.uint8:
        mask = (mask != 0).to(t.uint8)
    return mask.contiguous()


def _fracture_dev(mask, rects=True, stream=None):
    """Greedy fracture of a device mask on the GPU (lsopc_fracture_dev):
    (count, [(x, y, w, h), ...] or None)."""
    m = _device_u8(mask)
    H, W = m.shape
    sp = stream if stream is not None else nv.stream()
    count = ctypes.c_size_t()
    L = nv.lib()
    if not rects:
        nv.check(L.lsopc_fracture_dev(H, W, nv.ptr(m), None, 0, ctypes.byref(count), sp))
        return int(count.value), None
    cap = 1 << 16
    while True:
        buf = np.empty((cap, 4), dtype=np.int32)
        nv.check(L.lsopc_fracture_dev(H, W, nv.ptr(m), buf.ctypes.data_as(ctypes.c_void_p), cap,
                                      ctypes.byref(count), sp))
        if count.value <= cap:
            return int(count.value), [tuple(int(v) for v in r) for r in buf[:count.value]]
        cap = int(count.value)


def fracture(mask):
    """Greedy largest-rectangle decomposition, ties topmost then leftmost
    (metrics.py:55-104).  Returns [(x, y, w, h), ...].  A device (CUDA
    tensor) mask is fractured on the GPU."""
    if _is_device(mask):
        return _fracture_dev(mask)[1]
    m = _as_u8(mask)
    if m.ndim != 2:
        raise ValueError("mask must be 2-D")
    H, W = m.shape
    if m.size == 0:
        return []
    count = ctypes.c_size_t()
    nv.check(nv.lib().lsopc_fracture(H, W, m.ctypes.data_as(ctypes.c_void_p), None, 0,
                                     ctypes.byref(count)))
    buf = np.empty((max(count.value, 1), 4), dtype=np.int32)
    nv.check(nv.lib().lsopc_fracture(H, W, m.ctypes.data_as(ctypes.c_void_p),
                                     buf.ctypes.data_as(ctypes.c_void_p), count.value,
                                     ctypes.byref(count)))
    return [tuple(int(v) for v in r) for r in buf[:count.value]]


def _as_u8(mask):
    """The mask as contiguous bytes; the native fracture treats any non-zero
    byte as lit, so uint8 / bool masks pass through without a copy."""
    a = np.asarray(mask)
    if a.dtype == np.bool_:
        a = a.view(np.uint8)
    elif a.dtype != np.uint8:
        a = (a != 0).view(np.uint8)
    return np.ascontiguousarray(a)


def shot_count(mask):
    """len(fracture(mask)) (metrics.py:107-108); on the GPU for a device mask."""
    if _is_device(mask):
        return _fracture_dev(mask, rects=False)[0]
    m = _as_u8(mask)
    if m.ndim != 2:
        raise ValueError("mask must be 2-D")
    if m.size == 0:
        return 0
    count = ctypes.c_size_t()
    nv.check(nv.lib().lsopc_fracture(m.shape[0], m.shape[1], m.ctypes.data_as(ctypes.c_void_p),
                                     None, 0, ctypes.byref(count)))
    return int(count.value)


# ---------------------------------------------------------------------------
# EXTENSION: edge placement error (the reference has none; parity
# is UNPINNED -- checked against oracle/lsopc_oracle.py `epe` only)


@dataclass
class EPEReport:
    """EPE on the target's edges (ICCAD-2013 style): `samples` measured,
    `violations` with |EPE| > threshold, mean and max |EPE| (pixels; |EPE|
    saturates at threshold + 1)."""
    samples: int
    violations: int
    mean_abs: float
    max_abs: int
    spacing: int = 40
    threshold: int = 15

    def as_dict(self):
        return {"samples": self.samples, "violations": self.violations, "mean_abs": self.mean_abs,
                "max_abs": self.max_abs, "spacing": self.spacing, "threshold": self.threshold,
                "parity": "unpinned (no reference EPE)"}


def epe(printed, target, spacing=40, threshold=15, offset=None):
    """Edge placement error of a hard print against the target layout
    (lsopc_epe; see include/lsopc_b200.h for the definition): samples every
    `spacing` pixels on a lattice along the target's edges, the printed
    edge's signed displacement along the outward normal, violations where
    |EPE| > `threshold` (defaults: 40 / 15 px, the ICCAD-2013 nm figures at
    1 nm pitch).  Host or device uint8 / bool grids."""
    t = nv.torch()
    if offset is None:
        offset = spacing // 2

    def dev(a):
        if _is_device(a):
            return _device_u8(a)
        return nv.to_dev(np.not_equal(np.asarray(a), 0).view(np.uint8), np.uint8)

    p, g = dev(printed), dev(target)
    if tuple(p.shape) != tuple(g.shape) or p.dim() != 2:
        raise ValueError(f"dimension mismatch: {tuple(p.shape)} vs {tuple(g.shape)}")
    out = (ctypes.c_double * 4)()
    nv.check(nv.lib().lsopc_epe(p.shape[0], p.shape[1], nv.ptr(p), nv.ptr(g), int(spacing), int(offset),
                                int(threshold), int(threshold) + 1, out, nv.stream()))
    del t
    n = int(out[0])
    return EPEReport(samples=n, violations=int(out[1]), mean_abs=(out[2] / n if n else 0.0), max_abs=int(out[3]),
                     spacing=int(spacing), threshold=int(threshold))
