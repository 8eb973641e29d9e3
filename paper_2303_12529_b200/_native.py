"""ctypes binding of the C ABI in include/lsopc_b200.h, plus the device
plumbing (torch for device memory and streams).

There is no CPU fallback: importing the hot-path modules loads
`_lib/liblsopc_b200.so` and every operator raises if the library or a CUDA
device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DegenerateInputError, NumericalError

_LIB_PATH = Path(os.environ.get("LSOPC_B200_LIB") or
                 Path(__file__).resolve().parent / "_lib" / "liblsopc_b200.so")

OK, EINVAL, EDEGENERATE, ENUMERIC, ECUDA = 0, 1, 2, 3, 4
FP32, FP64 = 0, 1

EW = {"mask": 1, "heaviside": 2, "axpby": 3, "sigmoid": 4, "hard": 5, "neg": 6,
      "cg": 7, "motion": 8, "evolve": 9, "ahf": 10, "hypot": 11}
RD = {"sumsqdiff": 1, "dot": 2, "dotdiff": 3, "maxabs": 4, "countneq8": 5, "nonfinite": 6, "countneq": 7}


class LsopcConfig(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("curvature_weight", ctypes.c_double), ("sigma_z", ctypes.c_double),
                ("i_th", ctypes.c_double), ("eta", ctypes.c_double),
                ("d_upper", ctypes.c_double), ("d_lower", ctypes.c_double),
                ("max_iters", ctypes.c_int), ("stop_rel_tol", ctypes.c_double),
                ("stop_patience", ctypes.c_int), ("use_curvature", ctypes.c_int),
                ("cg_restart_every", ctypes.c_int), ("update_form", ctypes.c_int),
                ("skip_target_check", ctypes.c_int), ("grad_scheme", ctypes.c_int),
                ("reinit_every", ctypes.c_int)]


class LsopcResult(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("l2", ctypes.c_int), ("pvband", ctypes.c_int),
                ("nonfinite_iter", ctypes.c_int)]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_Z = ctypes.c_size_t

_SIGS = {
    "lsopc_last_error": (ctypes.c_char_p, []),
    "lsopc_abi_version": (_I, []),
    "lsopc_plan_create": (_I, [_I, _I, _I, ctypes.POINTER(_P)]),
    "lsopc_plan_destroy": (_I, [_P]),
    "lsopc_kset_create": (_I, [_P, _I, _I, _P, _P, _P, ctypes.POINTER(_P)]),
    "lsopc_kset_destroy": (_I, [_P]),
    "lsopc_kset_download": (_I, [_P, _P, _P]),
    "lsopc_aerial_intensity": (_I, [_P, _P, _P, _D, _P, _P]),
    "lsopc_print_corners": (_I, [_P, _P, _P, _P, _D, _D, _I, _P, _P, _P, _P]),
    "lsopc_socs_gradient": (_I, [_P, _P, _P, _P, _P, _D, _D, _P, _P]),
    "lsopc_convolve": (_I, [_P, _P, _P, _P, _P]),
    "lsopc_geometry_gradient": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lsopc_curvature": (_I, [_I, _I, _P, _P, _D, _P, _P]),
    "lsopc_tsdf": (_I, [_I, _I, _P, _D, _D, _P, _P]),
    "lsopc_elementwise": (_I, [_I, _Z, _P, _P, _D, _D, _D, _P, _P, _P]),
    "lsopc_reduce": (_I, [_I, _Z, _P, _P, _P, _P, ctypes.POINTER(_D), _P]),
    "lsopc_optimize": (_I, [_P, _P, _P, _P, _P, _P, ctypes.POINTER(LsopcConfig), _P, _P, _P,
                            ctypes.POINTER(LsopcResult), _P]),
    "lsopc_session_create": (_I, [_P, _P, _P, _P, _P, _P, ctypes.POINTER(LsopcConfig), _P,
                                  ctypes.POINTER(_P)]),
    "lsopc_session_enqueue": (_I, [_P, _I]),
    "lsopc_session_poll": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "lsopc_session_finish": (_I, [_P, _P, _P, _P, ctypes.POINTER(LsopcResult)]),
    "lsopc_session_phi": (_I, [_P, _P]),
    "lsopc_session_losses": (_I, [_P, _P, _P, _P]),
    "lsopc_session_destroy": (_I, [_P]),
    "lsopc_session_launches_per_iter": (_I, [_P]),
    "lsopc_fracture": (_I, [_I, _I, _P, _P, _Z, ctypes.POINTER(_Z)]),
    "lsopc_fracture_dev": (_I, [_I, _I, _P, _P, _Z, ctypes.POINTER(_Z), _P]),
    "lsopc_epe": (_I, [_I, _I, _P, _P, _I, _I, _I, _I, ctypes.POINTER(_D), _P]),
    "lsopc_session_time_passes": (_I, [_P, _I, ctypes.POINTER(_D)]),
    "lsopc_session_set_tile": (_I, [_P, _I, _I, _I, _I]),
    "lsopc_session_set_window": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I]),
    "lsopc_dsn_init": (_I, [_Z, _P, _P, _D, _D, _D, _P, _P, _P]),
    "lsopc_session_phase": (_I, [_P, _I]),
    "lsopc_session_scalars": (_P, [_P]),
    "lsopc_session_phi_ptr": (_P, [_P]),
    "lsopc_session_state_flag": (_P, [_P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the shared library (once).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise RuntimeError(
                    f"{_LIB_PATH} is missing: build it with "
                    "`python -m paper_2303_12529_b200.build` (no CPU fallback exists)")
            L = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc):
    if rc == OK:
        return
    msg = lib().lsopc_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EDEGENERATE:
        raise DegenerateInputError(msg)
    if rc == ENUMERIC:
        raise NumericalError(msg)
    raise RuntimeError(f"lsopc_b200 CUDA error: {msg}")


# ---------------------------------------------------------------------------
# device plumbing (torch owns device memory and the stream)

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        if not t.cuda.is_available():
            raise RuntimeError("lsopc_b200 needs a CUDA device (B200); no CPU fallback exists")
        _torch = t
    return _torch


def stream():
    return _P(torch().cuda.current_stream().cuda_stream)


_side = {}


def side_stream():
    """A second CUDA stream per (device, lane) for work that overlaps the
    lane's main stream (the final shot count overlaps the result copies)."""
    t = torch()
    key = (t.cuda.current_device(), lane())
    s = _side.get(key)
    if s is None:
        s = t.cuda.Stream()
        _side[key] = s
    return _P(s.cuda_stream)


def ptr(t):
    return _P(t.data_ptr()) if t is not None else None


def to_dev(a, dtype=np.float64):
    """Host array -> contiguous device tensor (copy)."""
    t = torch()
    arr = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    if not arr.flags.writeable:
        arr = arr.copy()
    return t.from_numpy(arr).to("cuda", non_blocking=False)


def empty(shape, dtype):
    t = torch()
    tdt = {np.float64: t.float64, np.uint8: t.uint8, np.complex128: t.complex128}[dtype]
    return t.empty(shape, dtype=tdt, device="cuda")


def to_host(t):
    return t.cpu().numpy()


_pinned = {}


def pinned_like(t):
    """A cached page-locked host tensor with t's shape and dtype (staging for
    fast device-to-host copies; callers copy out of it before reuse)."""
    key = (tuple(t.shape), t.dtype, lane())
    buf = _pinned.get(key)
    if buf is None:
        buf = torch().empty(t.shape, dtype=t.dtype, pin_memory=True)
        _pinned[key] = buf
    return buf


_h2d_done = {}


def to_dev_staged(a, dtype=np.uint8):
    """Host array -> new device tensor through a cached page-locked staging
    buffer (per shape, dtype and lane); an event guards the buffer against
    being overwritten while its previous upload is still in flight."""
    t = torch()
    arr = np.asarray(a, dtype=dtype)
    key = ("h2d", arr.shape, arr.dtype.str, lane())
    buf = _pinned.get(key)
    if buf is None:
        buf = t.from_numpy(np.empty(arr.shape, dtype=dtype)).pin_memory()
        _pinned[key] = buf
    done = _h2d_done.get(key)
    if done is not None:
        done.synchronize()
    np.copyto(buf.numpy(), arr)
    out = t.empty(arr.shape, dtype=buf.dtype, device="cuda")
    out.copy_(buf, non_blocking=True)
    ev = t.cuda.Event()
    ev.record()
    _h2d_done[key] = ev
    return out


# ---------------------------------------------------------------------------
# precision tiers

_PREC_NAMES = {"fp32": FP32, "fp64": FP64}
_default_precision = os.environ.get("LSOPC_B200_PRECISION", "fp64").lower()
if _default_precision not in _PREC_NAMES:
    raise ValueError(f"LSOPC_B200_PRECISION must be fp32 or fp64, got {_default_precision!r}")


def set_precision(name):
    """Select the transform precision for subsequent calls: "fp64" (exact
    drop-in, default) or "fp32" (complex64 transforms; level-set math stays
    float64)."""
    global _default_precision
    name = name.lower()
    if name not in _PREC_NAMES:
        raise ValueError(f"precision must be fp32 or fp64, got {name!r}")
    _default_precision = name


def get_precision():
    return _default_precision


def prec_code(name=None):
    return _PREC_NAMES[(name or _default_precision).lower()]


# ---------------------------------------------------------------------------
# plans (per grid shape and precision)


class Plan:
    def __init__(self, H, W, prec):
        self.H, self.W, self.prec = H, W, prec
        h = _P()
        check(lib().lsopc_plan_create(H, W, prec, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                lib().lsopc_plan_destroy(self.handle)
        except Exception:
            pass


_plans = {}
_tls = threading.local()


def set_lane(lane):
    """Select this thread's lane: work buffers (plans) and device spectra are
    kept per (shape, precision, lane), so threads on different lanes and
    different CUDA streams can run solves concurrently (parallel.py)."""
    _tls.lane = int(lane)


def lane():
    return getattr(_tls, "lane", 0)


def plan_for(shape, prec):
    H, W = int(shape[0]), int(shape[1])
    key = (H, W, prec, lane())
    p = _plans.get(key)
    if p is None:
        for n in (H, W):
            if n < 4 or n > 8192 or n & (n - 1):
                raise ValueError(
                    f"grid {W}x{H} unsupported: the transform supports power-of-two "
                    "sides in [4, 8192] (SPEC.md fields contract)")
        p = Plan(H, W, prec)
        _plans[key] = p
    return p


class DeviceKernelSet:
    """Device spectra of one KernelSet on one plan (litho.py:71-82 cache).
    `builds` counts spectra builds (K0) in this process."""

    builds = 0

    def __init__(self, plan, coeffs, weights):
        self.plan = plan
        c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.complex128))
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        h = _P()
        check(lib().lsopc_kset_create(plan.handle, c.shape[0], c.shape[1],
                                      c.ctypes.data_as(_P), w.ctypes.data_as(_P),
                                      stream(), ctypes.byref(h)))
        self.handle = h
        self.nk = c.shape[0]
        DeviceKernelSet.builds += 1

    def __del__(self):
        try:
            if self.handle:
                lib().lsopc_kset_destroy(self.handle)
        except Exception:
            pass


def elementwise(op, n, a=None, b=None, p0=0.0, p1=0.0, p2=0.0, out=None, out8=None):
    check(lib().lsopc_elementwise(EW[op], n, ptr(a), ptr(b), p0, p1, p2, ptr(out), ptr(out8),
                                  stream()))


def reduce(op, n, a=None, b=None, a8=None, b8=None):
    r = ctypes.c_double()
    check(lib().lsopc_reduce(RD[op], n, ptr(a), ptr(b), ptr(a8), ptr(b8), ctypes.byref(r),
                             stream()))
    return r.value
