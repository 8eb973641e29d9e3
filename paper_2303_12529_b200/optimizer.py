"""The DSO level-set ILT loop: drop-in for the reference `lsopc.optimizer`
(optimizer.py:1-341).

`optimize` runs the whole loop on the device through the C ABI
(`lsopc_optimize`): forward, losses, best iterate, adjoint, CG, CFL and the
level-set update are sm_100a kernels and the stop rule is evaluated on the
device, so the host only enqueues iterations and polls a flag.  The
operator-level functions (losses, gradients, CG, CFL, motion term) are the
same kernels exposed one call at a time.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nv
from . import litho
from .errors import DegenerateInputError
from .levelset import LevelSetField, heaviside, mask_from_phi
from .metrics import MetricsReport, shot_count

_EPS_GRAD = 1e-8

__all__ = [
    "OptConfig", "IterationRecord", "OptimizationResult",
    "ilt_loss", "pvb_loss", "ilt_gradient", "pvb_gradient",
    "velocity", "motion_term", "cfl_timestep", "cg_direction",
    "optimize", "modulation_search", "ModulationSearchResult",
]


@dataclass
class OptConfig:
    """Reference hyper-parameters and defaults (optimizer.py:38-64), plus
    `precision` ("fp64" | "fp32" | None = package default) selecting the
    transform tier.  epsilon and grid_side are accepted and inert, as in the
    reference."""
    alpha: float = 1.0
    beta: float = 7.5
    curvature_weight: float = 0.9
    sigma_z: float = 50.0
    i_th: float = 0.225
    epsilon: float = 0.03
    eta: float = 0.85
    d_upper: float = 900.0
    d_lower: float = -100.0
    max_iters: int = 100
    stop_rel_tol: float = 1e-4
    stop_patience: int = 5
    use_curvature: bool = True
    grid_side: int = 0
    cg_restart_every: int = 50
    precision: str = None
    # opt-in extensions, off by default (the reference has neither): the
    # Godunov upwind |grad phi| in the update term ("upwind") instead of the
    # central one (levelset.py:60-62), and phi <- tsdf(mask_from_phi(phi))
    # after every `reinit_every`-th completed iteration
    grad_scheme: str = "central"
    reinit_every: int = 0

    def __post_init__(self):
        if self.alpha < 0 or self.beta < 0 or (self.alpha == 0 and self.beta == 0):
            raise ValueError("alpha, beta must be >= 0 and not both zero")
        if not 0 < self.eta <= 1:
            raise ValueError("eta must be in (0, 1]")
        if self.sigma_z <= 0:
            raise ValueError("sigma_z must be positive")
        if self.max_iters < 0:
            raise ValueError("max_iters must be >= 0")
        if self.precision is not None and str(self.precision).lower() not in ("fp32", "fp64"):
            raise ValueError("precision must be fp32, fp64 or None")
        if self.grad_scheme not in ("central", "upwind"):
            raise ValueError("grad_scheme must be central or upwind")
        if self.reinit_every < 0:
            raise ValueError("reinit_every must be >= 0")


@dataclass
class IterationRecord:
    l_ilt: float
    l_pvb: float
    l_dso: float
    dt: float
    max_v: float
    max_step: float
    max_grad_mag: float


@dataclass
class OptimizationResult:
    final_mask: np.ndarray
    final_phi: LevelSetField
    metrics: MetricsReport
    loss_history: list
    iters_run: int
    wall_time: float


# ---------------------------------------------------------------------------
# operator-level API


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def _bcast_pair(a, b):
    a, b = np.broadcast_arrays(_f64(a), _f64(b))
    return np.ascontiguousarray(a), np.ascontiguousarray(b)


def ilt_loss(z, z_t):
    """sum (Z - Z_t)^2 (optimizer.py:88-90), deterministic device reduction."""
    a, b = _bcast_pair(z, z_t)
    if a.size == 0:
        return 0.0
    return float(nv.reduce("sumsqdiff", a.size, nv.to_dev(a), nv.to_dev(b)))


def pvb_loss(z_in, z_out, z_t):
    """sum (Z_in - Z_t)^2 + sum (Z_out - Z_t)^2 (optimizer.py:93-96)."""
    return float(ilt_loss(z_in, z_t) + ilt_loss(z_out, z_t))


def _socs_gradient_dev(mask, z, z_t, kernels, sigma_z, dose):
    m = _f64(mask)
    dks = litho.device_kernels(kernels, m.shape)
    zz, zt = _bcast_pair(z, z_t)
    out = nv.empty(m.shape, np.float64)
    md, zd, ztd = nv.to_dev(m), nv.to_dev(zz), nv.to_dev(zt)
    nv.check(nv.lib().lsopc_socs_gradient(dks.plan.handle, dks.handle, nv.ptr(md), nv.ptr(zd),
                                          nv.ptr(ztd), float(sigma_z), float(dose), nv.ptr(out),
                                          nv.stream()))
    return out


def _socs_gradient(mask, z, z_t, kernels, sigma_z, dose):
    """d sum (Z - Z_t)^2 / dM through the sigmoid and SOCS model
    (optimizer.py:99-111)."""
    return nv.to_host(_socs_gradient_dev(mask, z, z_t, kernels, sigma_z, dose))


def ilt_gradient(mask, z, z_t, kernels, cfg):
    """Nominal-corner loss gradient (optimizer.py:114-119)."""
    if kernels.side > min(np.shape(mask)):
        raise ValueError("kernel side exceeds grid")
    return _socs_gradient(mask, z, z_t, kernels, cfg.sigma_z, dose=1.0)


def pvb_gradient(mask, z_in, z_out, z_t, focus_kernels, defocus_kernels, cfg):
    """Inner (defocus, 0.98) + outer (focus, 1.02) gradients (optimizer.py:122-129)."""
    gi = _socs_gradient_dev(mask, z_in, z_t, defocus_kernels, cfg.sigma_z, litho.INNER.dose)
    go = _socs_gradient_dev(mask, z_out, z_t, focus_kernels, cfg.sigma_z, litho.OUTER.dose)
    out = nv.empty(gi.shape, np.float64)
    nv.elementwise("axpby", gi.numel(), gi, go, 1.0, 1.0, out=out)
    return nv.to_host(out)


def velocity(g_ilt, g_pvb, cfg):
    """alpha g_ilt + beta g_pvb (optimizer.py:132-134)."""
    a, b = _bcast_pair(g_ilt, g_pvb)
    out = nv.empty(a.shape, np.float64)
    if a.size:
        nv.elementwise("axpby", a.size, nv.to_dev(a), nv.to_dev(b), float(cfg.alpha),
                       float(cfg.beta), out=out)
    return nv.to_host(out)


def motion_term(v, phi, kappa=0.0):
    """-v |grad phi| + kappa (optimizer.py:137-140)."""
    from .levelset import gradient_magnitude
    gm = gradient_magnitude(phi)
    vv = np.ascontiguousarray(np.broadcast_to(_f64(v), gm.shape))
    out = nv.empty(gm.shape, np.float64)
    nv.elementwise("motion", gm.size, nv.to_dev(vv), nv.to_dev(gm), out=out)
    kk = np.ascontiguousarray(np.broadcast_to(_f64(kappa), gm.shape))
    res = nv.empty(gm.shape, np.float64)
    nv.elementwise("axpby", gm.size, out, nv.to_dev(kk), 1.0, 1.0, out=res)
    return nv.to_host(res)


def cfl_timestep(v_effective, eta):
    """(eta / max|v|, False), or (0, True) for a zero field (optimizer.py:143-151)."""
    a = np.ascontiguousarray(_f64(v_effective))
    vmax = float(nv.reduce("maxabs", a.size, nv.to_dev(a))) if a.size else 0.0
    if vmax == 0.0:
        return 0.0, True
    return eta / vmax, False


def cg_direction(g, g_prev=None, d_prev=None):
    """Polak-Ribiere+ direction with restart (optimizer.py:154-169)."""
    gg = np.ascontiguousarray(_f64(g))
    gd = nv.to_dev(gg)
    out = nv.empty(gg.shape, np.float64)
    beta = None
    if g_prev is not None and d_prev is not None and gg.size:
        gp = nv.to_dev(np.broadcast_to(_f64(g_prev), gg.shape))
        den = float(nv.reduce("dot", gg.size, gp, gp))
        if den != 0.0:
            b = float(nv.reduce("dotdiff", gg.size, gd, gp)) / den
            if b > 0.0:
                beta = b
    if beta is None:
        nv.elementwise("neg", gg.size, gd, out=out)
    else:
        dp = nv.to_dev(np.broadcast_to(_f64(d_prev), gg.shape))
        nv.elementwise("cg", gg.size, gd, dp, beta, out=out)
    return nv.to_host(out)


def _forward_losses(mask, target, focus_kernels, defocus_kernels, cfg):
    """optimizer.py:172-177."""
    prints = litho.print_corners(mask, focus_kernels, defocus_kernels, cfg, binarize=False)
    l_ilt = ilt_loss(prints.nominal, target)
    l_pvb = pvb_loss(prints.inner, prints.outer, target)
    return prints, l_ilt, l_pvb, cfg.alpha * l_ilt + cfg.beta * l_pvb


def _check_target(target):
    # one comparison pass (bool viewed as 0/1 bytes) and one count
    t = np.not_equal(np.asarray(target), 0).view(np.uint8)
    nz = int(np.count_nonzero(t))
    if nz == 0 or nz == t.size:
        raise DegenerateInputError("target layout is uniform")
    return t


# ---------------------------------------------------------------------------
# the loop


def _native_cfg(cfg, max_iters=None, stop_patience=None, use_curvature=None, update_form=0):
    c = nv.LsopcConfig()
    c.alpha, c.beta = float(cfg.alpha), float(cfg.beta)
    c.curvature_weight, c.sigma_z = float(cfg.curvature_weight), float(cfg.sigma_z)
    c.i_th, c.eta = float(cfg.i_th), float(cfg.eta)
    c.d_upper, c.d_lower = float(cfg.d_upper), float(cfg.d_lower)
    c.max_iters = int(cfg.max_iters if max_iters is None else max_iters)
    c.stop_rel_tol = float(cfg.stop_rel_tol)
    c.stop_patience = int(min(cfg.stop_patience if stop_patience is None else stop_patience, 2**31 - 1))
    c.use_curvature = int(bool(cfg.use_curvature if use_curvature is None else use_curvature))
    c.cg_restart_every = int(cfg.cg_restart_every)
    c.update_form = int(update_form)
    c.grad_scheme = 1 if getattr(cfg, "grad_scheme", "central") == "upwind" else 0
    c.reinit_every = int(getattr(cfg, "reinit_every", 0))
    return c


def _precision(cfg):
    """The transform tier of a config; reference OptConfigs have no
    `precision` field and take the package default."""
    return getattr(cfg, "precision", None)


def _check_kernel_sets(shape, focus_kernels, defocus_kernels):
    for ks, sel in ((focus_kernels, "focus"), (defocus_kernels, "defocus")):
        if ks.side > min(shape):
            raise ValueError(f"kernel side {ks.side} exceeds grid {shape}")
        if ks.condition != sel:
            raise ValueError(f"kernel set condition {ks.condition!r} does not match "
                             f"process condition {sel!r}")


def _target_bytes(target):
    """The target as contiguous uint8 bytes without a host pass when it
    already is uint8 / bool (the device binarises it); other dtypes are
    binarised here."""
    t = np.asarray(target)
    if t.ndim != 2:
        raise ValueError("target must be a 2-D layout")
    if t.dtype == np.bool_:
        t = t.view(np.uint8)
    elif t.dtype != np.uint8:
        t = np.not_equal(t, 0).view(np.uint8)
    return np.ascontiguousarray(t)


def _prepare(target, focus_kernels, defocus_kernels, cfg, phi0, modulation, scan=True):
    """Validation of optimize's inputs (optimizer.py:197-228).  scan=False
    leaves the uniform-target check to the device (lsopc_session_create)."""
    target = _check_target(target) if scan else _target_bytes(target)
    shape = target.shape
    if phi0 is not None and phi0.shape != shape:
        raise ValueError("phi0 dimensions do not match target")
    m = None
    if modulation is not None:
        m = _f64(modulation)
        if m.shape != shape:
            raise ValueError("modulation dimensions do not match target")
        if m.size and (m.min() < 0 or m.max() > 1):
            raise ValueError("modulation values must lie in [0, 1]")
    _check_kernel_sets(shape, focus_kernels, defocus_kernels)
    prec = _precision(cfg)
    fk = litho.device_kernels(focus_kernels, shape, prec)
    dk = litho.device_kernels(defocus_kernels, shape, prec)
    return target, m, fk, dk


def _is_device_tensor(x):
    return x is not None and hasattr(x, "is_cuda") and x.is_cuda


def _device_f64(x, shape, what):
    if x is None:
        return None
    if tuple(x.shape) != tuple(shape):
        raise ValueError(f"{what} dimensions do not match target")
    return x.to(dtype=nv.torch().float64).contiguous()


def _device_inputs(target, focus_kernels, defocus_kernels, cfg, phi0, modulation):
    """`_prepare` for a device-resident initial state (DevelSet-Net front end,
    dsn.py, which has already clipped phi0 and mapped m through the AHF on the
    device).  The other input may be a host array / LevelSetField: it is
    validated like `optimize` validates it (optimizer.py:215-228) and
    uploaded, so mixed input kinds behave like all-host ones."""
    target = _check_target(target)
    shape = target.shape
    _check_kernel_sets(shape, focus_kernels, defocus_kernels)
    if phi0 is not None and not _is_device_tensor(phi0):
        p = phi0.phi if hasattr(phi0, "phi") else _f64(phi0)
        if p.shape != shape:
            raise ValueError("phi0 dimensions do not match target")
        phi0 = nv.to_dev(p)
    if modulation is not None and not _is_device_tensor(modulation):
        m = _f64(modulation)
        if m.shape != shape:
            raise ValueError("modulation dimensions do not match target")
        if m.size and (m.min() < 0 or m.max() > 1):
            raise ValueError("modulation values must lie in [0, 1]")
        modulation = nv.to_dev(m)
    prec = _precision(cfg)
    fk = litho.device_kernels(focus_kernels, shape, prec)
    dk = litho.device_kernels(defocus_kernels, shape, prec)
    return target, fk, dk, _device_f64(phi0, shape, "phi0"), _device_f64(modulation, shape, "modulation")


def _optimize_device(target, focus_kernels, defocus_kernels, cfg, phi0=None, modulation=None, shots_on="device"):
    """Device part of `optimize`: the loop, final prints and the device-to-host
    copies.  Returns the pieces `_assemble` turns into an OptimizationResult
    (split so a batch driver can overlap one clip's host tail with the next
    clip's device loop).  shots_on="host": batch drivers, whose next clip's
    persistent passes hold every SM, count shots with the host implementation
    on a tail thread instead of the device kernel (one thread-block cluster
    that would otherwise wait for, and then delay, those passes)."""
    t0 = time.perf_counter()
    if _is_device_tensor(phi0) or _is_device_tensor(modulation):
        target, fk, dk, p0, mdv = _device_inputs(target, focus_kernels, defocus_kernels, cfg, phi0, modulation)
    else:
        target, m, fk, dk = _prepare(target, focus_kernels, defocus_kernels, cfg, phi0, modulation, scan=False)
        p0 = nv.to_dev(phi0.phi) if phi0 is not None else None
        mdv = nv.to_dev(m) if m is not None else None
    shape = target.shape
    # the raw bytes go up; the device binarises them (target != 0) and
    # rejects a uniform target (optimizer.py:197-201) in lsopc_session_create
    td = nv.to_dev_staged(target, np.uint8)
    best = nv.empty(shape, np.float64)
    fmask = nv.empty(shape, np.uint8)
    hist = np.zeros((cfg.max_iters + 1, 7))
    res = nv.LsopcResult()
    c = _native_cfg(cfg)
    nv.check(nv.lib().lsopc_optimize(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), nv.ptr(p0),
                                     nv.ptr(mdv), ctypes.byref(c), nv.ptr(best), nv.ptr(fmask),
                                     hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res),
                                     nv.stream()))
    # wall_time is taken before the shot count, as in the reference
    # (optimizer.py:274-281).  The shot count of the final mask runs on the GPU
    # (one thread-block cluster, on a side stream driven by a helper thread;
    # the ctypes call releases the GIL) while the mask and the float64 phi are
    # copied straight into page-locked host tensors from torch's caching host
    # allocator, whose numpy views are the returned arrays (no host-side copy).
    if shots_on == "device":
        shots = _tail_pool().submit(_device_shots, fmask, nv.side_stream())
    t = nv.torch()
    mask_h = t.empty(shape, dtype=t.uint8, pin_memory=True)
    phi_h = t.empty(shape, dtype=t.float64, pin_memory=True)
    mask_h.copy_(fmask, non_blocking=True)
    phi_h.copy_(best, non_blocking=True)
    t.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    if shots_on != "device":
        shots = _tail_pool().submit(shot_count, mask_h.numpy())
    return mask_h.numpy(), phi_h.numpy(), (res.iters, res.l2, res.pvband), hist, wall, shots


_TAIL = None


def _device_shots(fmask, stream):
    from .metrics import _fracture_dev
    return _fracture_dev(fmask, rects=False, stream=stream)[0]


def _tail_pool():
    global _TAIL
    if _TAIL is None:
        from concurrent.futures import ThreadPoolExecutor
        _TAIL = ThreadPoolExecutor(max_workers=4, thread_name_prefix="lsopc-tail")
    return _TAIL


def _assemble(parts, cfg, phi0=None):
    """Host tail of `optimize`: shot count, history records, result."""
    final_mask, best_phi, (iters, l2, pvb), hist, wall, shots = parts
    shots = shots.result() if hasattr(shots, "result") else shot_count(final_mask)
    history = [IterationRecord(*(float(v) for v in row)) for row in hist[:iters]]
    bounds = (cfg.d_upper, cfg.d_lower)
    if phi0 is not None and not _is_device_tensor(phi0):
        # the initial iterate keeps phi0's own bounds (optimizer.py:219-220,231);
        # the best iterate is the first strict minimum of the recorded losses
        losses = [h.l_dso for h in history]
        if not losses or int(np.argmin(losses)) == 0:
            bounds = (phi0.d_upper, phi0.d_lower)
    report = MetricsReport(l2=l2, pvband=pvb, shots=shots, wall_time=wall, iters=iters)
    return OptimizationResult(final_mask=final_mask,
                              final_phi=LevelSetField(best_phi, bounds[0], bounds[1]),
                              metrics=report, loss_history=history, iters_run=iters,
                              wall_time=wall)


def optimize(target, focus_kernels, defocus_kernels, cfg, phi0=None, modulation=None):
    """Full level-set ILT loop on the device (optimizer.py:204-284).  Returns
    the lowest-loss iterate, binarised, with hard-resist metrics and the loss
    history."""
    parts = _optimize_device(target, focus_kernels, defocus_kernels, cfg, phi0, modulation)
    return _assemble(parts, cfg, phi0)


@dataclass
class ModulationSearchResult:
    m_gt: np.ndarray
    best_delta_h: float
    candidates: list = field(default_factory=list)


def modulation_offsets(num_samples):
    """Candidate shifts delta_h of modulation_search (optimizer.py:306-307)."""
    if num_samples < 1:
        raise ValueError("num_samples must be >= 1")
    return [0.0] if num_samples == 1 else list(np.linspace(-20.0, 20.0, num_samples))


def modulation_eval_cfg(cfg):
    """The search's evaluation config: curvature on (optimizer.py:308)."""
    return OptConfig(**{**cfg.__dict__, "use_curvature": True})


def modulation_score(phi_gt, target, focus_kernels, defocus_kernels, eval_cfg, dh, eval_steps=10, resident=None):
    """Final L_DSO of one candidate gate H(phi_gt + dh) (optimizer.py:312-336):
    `eval_steps` device iterations from phi_gt with curvature gated by it
    (CFL break, no patience rule), then the forward losses of the last
    iterate, all on the device (lsopc_session_losses).  `resident` (a dict
    owned by the caller, one per stream) keeps phi_gt and the target on the
    device across candidates; the gate is formed there."""
    import torch
    key = (id(phi_gt), id(target))
    target, _, fk, dk = _prepare(target, focus_kernels, defocus_kernels, eval_cfg, phi_gt, None)
    res = resident if resident is not None else {}
    if res.get("key") != key:
        res.update(key=key, td=nv.to_dev(target, np.uint8), pd=nv.to_dev(phi_gt.phi))
    gate = ((res["pd"] + float(dh)) >= 0.0).to(torch.float64)  # levelset.py:142-144 on phi_gt + dh
    c = _native_cfg(eval_cfg, max_iters=eval_steps, stop_patience=2**31 - 1, use_curvature=True, update_form=1)
    L = nv.lib()
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(res["td"]), nv.ptr(res["pd"]),
                                    nv.ptr(gate), ctypes.byref(c), nv.stream(), ctypes.byref(sess)))
    try:
        if eval_steps > 0:
            nv.check(L.lsopc_session_enqueue(sess, eval_steps))
        l_dso = ctypes.c_double()
        nv.check(L.lsopc_session_losses(sess, None, None, ctypes.byref(l_dso)))
    finally:
        L.lsopc_session_destroy(sess)
    return float(l_dso.value)


def modulation_pick(phi_gt, candidates, gate=None):
    """Best candidate, ties on smallest |dh| then dh (optimizer.py:338-341);
    m_gt = gate(phi_gt + best_dh), the device Heaviside by default."""
    best_loss = min(l for _, l in candidates)
    tied = [dh for dh, l in candidates if l == best_loss]
    best_dh = min(tied, key=lambda d: (abs(d), d))
    m_gt = (gate or heaviside)(phi_gt.phi + best_dh).astype(np.float64)
    return ModulationSearchResult(m_gt, best_dh, list(candidates))


def modulation_search(phi_gt, target, focus_kernels, defocus_kernels, cfg, num_samples=41,
                      eval_steps=10):
    """Exhaustive curvature-gate search (optimizer.py:294-341): each candidate
    gate H(phi_gt + dh) is scored by L_DSO after `eval_steps` device
    iterations with curvature on; ties break on smallest |dh|, then dh.
    `parallel.modulation_search_sharded` spreads the candidates over GPUs."""
    offsets = modulation_offsets(num_samples)
    target = _check_target(target)
    eval_cfg = modulation_eval_cfg(cfg)
    resident = {}
    candidates = [(dh, modulation_score(phi_gt, target, focus_kernels, defocus_kernels, eval_cfg, dh, eval_steps,
                                        resident)) for dh in offsets]
    return modulation_pick(phi_gt, candidates)
