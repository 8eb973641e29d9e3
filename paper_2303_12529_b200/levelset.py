"""Level-set machinery: drop-in for the reference `lsopc.levelset`
(levelset.py:1-166).  TSDF, mask conversion, stencils, curvature, Heaviside
and the explicit step run on the device (bit-identical float64 arithmetic);
`extract_boundaries` is a host helper off the optimisation path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as nv
from .errors import DegenerateInputError, NumericalError

D_UPPER_DEFAULT = 900.0
D_LOWER_DEFAULT = -100.0
EPS_DEN = 1e-8

__all__ = [
    "LevelSetField", "GeometryGradient",
    "extract_boundaries", "tsdf_from_mask", "mask_from_phi",
    "geometry_gradient", "gradient_magnitude", "curvature",
    "heaviside", "ahf", "evolve_step",
]


@dataclass
class LevelSetField:
    """phi (<= 0 inside) with truncation bounds D_l < 0 < D_u (levelset.py:31-49)."""
    phi: np.ndarray
    d_upper: float = D_UPPER_DEFAULT
    d_lower: float = D_LOWER_DEFAULT

    def __post_init__(self):
        self.phi = np.asarray(self.phi, dtype=np.float64)
        if not (self.d_lower < 0.0 < self.d_upper):
            raise ValueError(
                f"truncation bounds must satisfy D_l < 0 < D_u, got [{self.d_lower}, {self.d_upper}]")

    @property
    def shape(self):
        return self.phi.shape

    def copy(self):
        return LevelSetField(self.phi.copy(), self.d_upper, self.d_lower)


@dataclass
class GeometryGradient:
    """First and second central differences of phi (levelset.py:52-62)."""
    gx: np.ndarray
    gy: np.ndarray
    gxx: np.ndarray
    gyy: np.ndarray
    gxy: np.ndarray
    _mag: np.ndarray = field(default=None, repr=False, compare=False)

    @property
    def magnitude(self):
        if self._mag is None:
            gx = np.asarray(self.gx, dtype=np.float64)
            gy = np.asarray(self.gy, dtype=np.float64)
            if gx.size == 0:
                return np.hypot(gx, gy)
            out = nv.empty(gx.shape, np.float64)
            nv.elementwise("hypot", gx.size, nv.to_dev(gx), nv.to_dev(gy), out=out)
            self._mag = nv.to_host(out)
        return self._mag


def _phi_array(phi):
    return phi.phi if isinstance(phi, LevelSetField) else np.asarray(phi, dtype=np.float64)


def _as_2d(a):
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D field, got shape {a.shape}")
    return a


def extract_boundaries(mask):
    """(b_h, b_v): pixels differing from their up/down (b_h) or left/right
    (b_v) neighbour, zero padding outside (levelset.py:69-83)."""
    p = np.pad(np.asarray(mask, dtype=np.uint8), 1, mode="constant")
    c = p[1:-1, 1:-1]
    b_h = ((c ^ p[:-2, 1:-1]) | (c ^ p[2:, 1:-1])).astype(np.uint8)
    b_v = ((c ^ p[1:-1, :-2]) | (c ^ p[1:-1, 2:])).astype(np.uint8)
    return b_h, b_v


def tsdf_from_mask(mask, d_upper=D_UPPER_DEFAULT, d_lower=D_LOWER_DEFAULT):
    """Truncated signed distance: -(d - 1/2) inside, d - 1/2 outside, d the
    distance to the nearest opposite-phase pixel centre (levelset.py:86-101);
    exact EDT on the device."""
    m = _as_2d(np.asarray(mask))
    lit = (m != 0).astype(np.uint8)
    if lit.all() or not lit.any():
        raise DegenerateInputError("mask is uniform: no boundary exists")
    if not (d_lower < 0.0 < d_upper):
        raise ValueError(
            f"truncation bounds must satisfy D_l < 0 < D_u, got [{d_lower}, {d_upper}]")
    md = nv.to_dev(lit, np.uint8)
    out = nv.empty(m.shape, np.float64)
    nv.check(nv.lib().lsopc_tsdf(m.shape[0], m.shape[1], nv.ptr(md), float(d_upper),
                                 float(d_lower), nv.ptr(out), nv.stream()))
    return LevelSetField(nv.to_host(out), d_upper, d_lower)


def _threshold(phi, op):
    a = _phi_array(phi)
    if a.size == 0:
        return np.zeros(a.shape, dtype=np.uint8)
    out = nv.empty(a.shape, np.uint8)
    nv.elementwise(op, a.size, nv.to_dev(a), out8=out)
    return nv.to_host(out)


def mask_from_phi(phi):
    """1 where phi <= 0 (levelset.py:104-106)."""
    return _threshold(phi, "mask")


def geometry_gradient(phi):
    """Central differences with replicate padding (levelset.py:109-119)."""
    a = _as_2d(_phi_array(phi))
    H, W = a.shape
    d = nv.to_dev(a)
    outs = [nv.empty(a.shape, np.float64) for _ in range(6)]
    nv.check(nv.lib().lsopc_geometry_gradient(H, W, nv.ptr(d), *(nv.ptr(o) for o in outs),
                                              nv.stream()))
    gx, gy, gxx, gyy, gxy, mag = (nv.to_host(o) for o in outs)
    return GeometryGradient(gx, gy, gxx, gyy, gxy, _mag=mag)


def gradient_magnitude(phi):
    a = _as_2d(_phi_array(phi))
    d = nv.to_dev(a)
    out = nv.empty(a.shape, np.float64)
    nv.check(nv.lib().lsopc_geometry_gradient(a.shape[0], a.shape[1], nv.ptr(d), None, None, None,
                                              None, None, nv.ptr(out), nv.stream()))
    return nv.to_host(out)


def curvature(phi, m=None, weight=1.0):
    """kappa = weight * m * (gxx gy^2 - 2 gx gy gxy + gyy gx^2) / (gx^2 + gy^2 + 1e-8)
    (levelset.py:126-139)."""
    a = _as_2d(_phi_array(phi))
    d = nv.to_dev(a)
    md = None
    if m is not None:
        mm = np.broadcast_to(np.asarray(m, dtype=np.float64), a.shape)
        md = nv.to_dev(mm)
    out = nv.empty(a.shape, np.float64)
    nv.check(nv.lib().lsopc_curvature(a.shape[0], a.shape[1], nv.ptr(d), nv.ptr(md), float(weight),
                                      nv.ptr(out), nv.stream()))
    return nv.to_host(out)


def heaviside(phi):
    """1 where phi >= 0 (levelset.py:142-144)."""
    return _threshold(phi, "heaviside")


def ahf(phi, epsilon=0.03):
    """0.5 (1 + (2/pi) arctan(phi / epsilon)) (levelset.py:147-151)."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    a = _phi_array(phi)
    if a.size == 0:
        return np.zeros(a.shape)
    out = nv.empty(a.shape, np.float64)
    nv.elementwise("ahf", a.size, nv.to_dev(a), p0=float(epsilon), out=out)
    return nv.to_host(out)


def evolve_step(lsf, dphi_dt, dt):
    """phi <- clamp(phi + dt * dphi_dt, D_l, D_u) (levelset.py:154-166)."""
    if dt <= 0:
        raise ValueError("time step must be positive")
    upd = np.asarray(dphi_dt, dtype=np.float64)
    if upd.shape != lsf.phi.shape:
        raise ValueError("update field dimensions do not match phi")
    ud = nv.to_dev(upd)
    r = nv.reduce("nonfinite", upd.size, ud) if upd.size else 0.0
    if r > 0:
        idx = upd.size - int(r)
        y, x = np.unravel_index(idx, upd.shape)
        raise NumericalError(f"non-finite update at pixel (x={x}, y={y})")
    out = nv.empty(upd.shape, np.float64)
    nv.elementwise("evolve", upd.size, nv.to_dev(lsf.phi), ud, p0=float(dt),
                   p1=float(lsf.d_lower), p2=float(lsf.d_upper), out=out)
    return LevelSetField(nv.to_host(out), lsf.d_upper, lsf.d_lower)
