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

__all__ = ["MetricsReport", "l2_error", "pvband", "fracture", "shot_count"]


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
