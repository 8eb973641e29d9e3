"""Oversized tile split across ranks (BASELINE configs[4]).

The reference optimises one periodic N x N tile with circular FFTs
(`fields.py:5-6`, `litho.py:114-126`).  Here the tile is cut into strips, one
per rank: full-width strips of rows (axis=0, the default) or full-height
strips of columns (axis=1).  Each rank runs the unchanged device pipeline on
a power-of-two window that holds its interior lines plus halos of at least
HALO = 2 * (K // 2) lines on each side (the forward field at a pixel needs
the mask within +-K//2, the adjoint within +-2 * (K//2)), so every interior
value equals the full-tile computation.  Row strips are the default because
the window's long (tile-length, 8192-point) axis then lies along the rows,
whose transforms stream by TMA: an 2048 x 8192 window iterates in 10.6 ms
against 20.3 ms for the 8192 x 2048 column window (scripts/tile_passes.py).
Per iteration:

    phase 0  forward on the window                -> all_reduce(sum)  losses
    phase 1  stop rule, adjoint, CG dot partials  -> all_reduce(sum)  dots
    phase 2  CG direction, level-set velocity     -> all_reduce(max)  |v|, |grad phi|
    phase 3  CFL step, interior update            -> all_reduce(max)  step
    phase 4  history record
    halo     exchange HALO columns of phi with both neighbours (wrapping)

Optics wrap around the tile edge (periodic, like the reference's FFT); the
phi stencil uses replicate padding at the global left/right edge
(`levelset.py:112`), so the edge ranks clamp their stencil to the interior.
Losses, dots, maxima and the final L2/PVB are summed over interiors only.
All ranks see the same scalars, so the stop rule, best iterate and CG
restarts agree everywhere.

Collectives go through `torch.distributed` on the default group: NCCL keeps
them on the stream; with gloo (CPU tests, several ranks sharing one GPU) the
small buffers are staged through host memory.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nv
from . import litho
from .levelset import LevelSetField
from .metrics import MetricsReport, shot_count


@dataclass
class Strip:
    """Geometry of one rank's strip along the split axis (1: columns, the
    tile of H x W cut into full-height strips; 0: rows, full-width strips,
    described here in the transposed frame, so `W` is the tile's extent along
    the split axis and `H` the other one): interior [x0, x1) of the global
    tile, window width ww whose line c is global line (x0 - hl + c) mod W."""
    rank: int
    world: int
    H: int
    W: int
    x0: int
    x1: int
    ww: int
    hl: int
    halo: int
    axis: int = 1

    @property
    def interior(self):
        return self.hl, self.hl + (self.x1 - self.x0)

    def columns(self):
        """Global line (column for axis 1, row for axis 0) of every window line."""
        return (self.x0 - self.hl + np.arange(self.ww)) % self.W

    lines = columns

    def stencil_bounds(self):
        """Neighbour clamp of the phi stencil along the split axis, window coordinates."""
        i0, i1 = self.interior
        return (i0 if self.rank == 0 else 0), (i1 if self.rank == self.world - 1 else self.ww)

    @property
    def window_shape(self):
        return (self.H, self.ww) if self.axis == 1 else (self.ww, self.H)


def strip_geometry(H, W, world, rank, K, axis=1):
    """Strips of equal width along `axis` (1: columns, 0: rows) of an H x W
    tile; windows are powers of two along the split axis."""
    if axis not in (0, 1):
        raise ValueError("axis must be 0 (row strips) or 1 (column strips)")
    if axis == 0:
        H, W = W, H  # describe row strips in the transposed frame
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if W % world:
        raise ValueError(f"tile extent {W} is not divisible by {world} ranks")
    halo = 2 * (K // 2)
    wi = W // world
    x0 = rank * wi
    if world == 1:
        return Strip(rank, world, H, W, 0, W, W, 0, halo, axis)
    if halo > wi:
        raise ValueError(f"strip width {wi} is narrower than the halo {halo}")
    if wi + 2 * halo > W:
        raise ValueError(f"{world} strips of a {W}-wide tile cannot carry {halo}-line halos")
    ww = 1
    while ww < wi + 2 * halo:
        ww *= 2
    ww = min(ww, W)  # at most the whole tile (then the window wraps onto itself)
    hl = (ww - wi) // 2
    return Strip(rank, world, H, W, x0, x0 + wi, ww, hl, halo, axis)


class _CudaView:
    """Zero-copy torch view of a device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _dist():
    import torch.distributed as dist
    return dist


def _backend_is_nccl():
    dist = _dist()
    return dist.is_initialized() and dist.get_backend() == "nccl"


def all_reduce_(t, op):
    """In-place all-reduce of a small device tensor (staged on the host for gloo)."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    if _backend_is_nccl():
        dist.all_reduce(t, op=op)
    else:
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    return t


def exchange_halos(phi, strip, tags=True):
    """Refresh the HALO columns on each side of the interior of `phi`
    (H x ww torch tensor) from the neighbouring ranks' interiors (wrapping).

    NCCL ignores P2P tags and pairs the operations between two ranks by
    position, so the order below is what keeps the two messages apart when
    left == right (two ranks): each rank sends its left edge first and its
    right edge second, and receives from its right neighbour first (that
    neighbour's left edge) and from its left neighbour second.  With distinct
    neighbours the order is immaterial.  `tags=False` exercises that
    positional matching on backends that honour tags (gloo)."""
    dist = _dist()
    if strip.world == 1:
        return
    import torch
    h = strip.halo
    i0, i1 = strip.interior
    left, right = (strip.rank - 1) % strip.world, (strip.rank + 1) % strip.world
    nccl = _backend_is_nccl()
    stage = (lambda t: t) if nccl else (lambda t: t.cpu())
    if strip.axis == 0:  # row strips: halo rows are contiguous
        phi = phi.t()
    send_l = stage(phi[:, i0:i0 + h].contiguous())    # -> left neighbour's right halo
    send_r = stage(phi[:, i1 - h:i1].contiguous())    # -> right neighbour's left halo
    recv_l = torch.empty_like(send_l)
    recv_r = torch.empty_like(send_r)
    t1, t2 = (1, 2) if tags else (0, 0)
    ops = [dist.P2POp(dist.isend, send_l, left, tag=t1), dist.P2POp(dist.isend, send_r, right, tag=t2),
           dist.P2POp(dist.irecv, recv_r, right, tag=t1), dist.P2POp(dist.irecv, recv_l, left, tag=t2)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    phi[:, i0 - h:i0].copy_(recv_l)
    phi[:, i1:i1 + h].copy_(recv_r)


@dataclass
class TiledResult:
    final_mask: np.ndarray      # global tile (every rank)
    final_phi: LevelSetField    # global tile (every rank)
    metrics: MetricsReport
    loss_history: list
    iters_run: int
    wall_time: float
    loop_time: float = 0.0      # seconds in the iteration loop (device-synchronised)


def optimize_tiled(target, focus_kernels, defocus_kernels, cfg, phi0=None, axis=0):
    """`optimize` (optimizer.py:204-284) of one tile split into strips over
    the ranks of the default process group (a single process runs the whole
    tile as one strip).  Every rank passes the same global `target` (and
    `phi0`); every rank returns the assembled global result.  axis=0: strips
    of rows (full width), axis=1: strips of columns (full height)."""
    import time
    import torch
    from .optimizer import IterationRecord, _check_target, _native_cfg

    t0 = time.perf_counter()
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    target = _check_target(target)
    H, W = target.shape
    st = strip_geometry(H, W, world, rank, focus_kernels.side, axis)
    lines = st.lines()
    i0, i1 = st.interior
    lo, hi = st.stencil_bounds()
    wshape = st.window_shape
    prec = getattr(cfg, "precision", None)

    def window(a):  # the window's lines of a global (host or device) array
        return a[:, lines] if axis == 1 else a[lines, :]

    # initial level set: the whole tile's TSDF (levelset.py:86-101) or phi0, windowed
    if phi0 is None:
        td_full = nv.to_dev(target, np.uint8)
        phi_full = nv.empty((H, W), np.float64)
        nv.check(nv.lib().lsopc_tsdf(H, W, nv.ptr(td_full), float(cfg.d_upper), float(cfg.d_lower),
                                     nv.ptr(phi_full), nv.stream()))
        idx = torch.as_tensor(lines, device=phi_full.device)
        phi_win = (phi_full[:, idx] if axis == 1 else phi_full[idx, :]).contiguous()
        del phi_full, td_full
    else:
        p = np.asarray(phi0.phi, dtype=np.float64)
        if p.shape != target.shape:
            raise ValueError("phi0 dimensions do not match target")
        phi_win = nv.to_dev(np.ascontiguousarray(window(p)))
    tgt_win = nv.to_dev(np.ascontiguousarray(window(target)), np.uint8)

    fk = litho.device_kernels(focus_kernels, wshape, prec)
    dk = litho.device_kernels(defocus_kernels, wshape, prec)
    c = _native_cfg(cfg)
    c.skip_target_check = 1
    L = nv.lib()
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(tgt_win), nv.ptr(phi_win), None,
                                    ctypes.byref(c), nv.stream(), ctypes.byref(sess)))
    try:
        if axis == 1:
            nv.check(L.lsopc_session_set_window(sess, i0, i1, lo, hi, 0, H, 0, H))
        else:
            nv.check(L.lsopc_session_set_window(sess, 0, W, 0, W, i0, i1, lo, hi))
        sc = torch.as_tensor(_CudaView(L.lsopc_session_scalars(sess), (8,), "<f8"), device="cuda")
        phi = torch.as_tensor(_CudaView(L.lsopc_session_phi_ptr(sess), wshape, "<f8"), device="cuda")
        flag = torch.as_tensor(_CudaView(L.lsopc_session_state_flag(sess), (1,), "<i4"), device="cuda")
        SUM, MAX = dist.ReduceOp.SUM, dist.ReduceOp.MAX
        torch.cuda.synchronize()
        t_loop = time.perf_counter()
        # The device stop flag turns every later phase into a no-op (its
        # bodies check it), so the host reads it only every `poll` iterations
        # and the stream stays queued in between; it is identical on every
        # rank (same global scalars), so all ranks leave together.
        poll = 4
        for i in range(cfg.max_iters):
            nv.check(L.lsopc_session_phase(sess, 0))
            all_reduce_(sc[0:2], SUM)
            nv.check(L.lsopc_session_phase(sess, 1))
            all_reduce_(sc[2:4], SUM)
            nv.check(L.lsopc_session_phase(sess, 2))
            all_reduce_(sc[4:6], MAX)
            nv.check(L.lsopc_session_phase(sess, 3))
            all_reduce_(sc[6:7], MAX)
            nv.check(L.lsopc_session_phase(sess, 4))
            if (i + 1) % poll == 0 and int(flag.item()):
                break
            exchange_halos(phi, st)
        torch.cuda.synchronize()
        t_loop = time.perf_counter() - t_loop
        best = nv.empty(wshape, np.float64)
        fmask = nv.empty(wshape, np.uint8)
        hist = np.zeros((cfg.max_iters + 1, 7))
        res = nv.LsopcResult()
        nv.check(L.lsopc_session_finish(sess, nv.ptr(best), nv.ptr(fmask), hist.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.byref(res)))
    finally:
        L.lsopc_session_destroy(sess)
    counts = torch.tensor([float(res.l2), float(res.pvband)], dtype=torch.float64, device="cuda")
    all_reduce_(counts, dist.ReduceOp.SUM)
    # assemble the global mask and phi from every rank's interior
    my_mask = (fmask[:, i0:i1] if axis == 1 else fmask[i0:i1, :]).contiguous()
    my_phi = (best[:, i0:i1] if axis == 1 else best[i0:i1, :]).contiguous()
    if world > 1:
        if _backend_is_nccl():
            masks = [torch.empty_like(my_mask) for _ in range(world)]
            phis = [torch.empty_like(my_phi) for _ in range(world)]
            dist.all_gather(masks, my_mask)
            dist.all_gather(phis, my_phi)
            masks = [m.cpu().numpy() for m in masks]
            phis = [p.cpu().numpy() for p in phis]
        else:
            masks = [None] * world
            phis = [None] * world
            dist.all_gather_object(masks, my_mask.cpu().numpy())
            dist.all_gather_object(phis, my_phi.cpu().numpy())
        final_mask = np.concatenate(masks, axis=axis)
        final_phi = np.concatenate(phis, axis=axis)
    else:
        final_mask = my_mask.cpu().numpy()
        final_phi = my_phi.cpu().numpy()
    wall = time.perf_counter() - t0
    history = [IterationRecord(*(float(v) for v in row)) for row in hist[:res.iters]]
    report = MetricsReport(l2=int(counts[0].item()), pvband=int(counts[1].item()), shots=shot_count(final_mask),
                           wall_time=wall, iters=res.iters)
    return TiledResult(final_mask=final_mask, final_phi=LevelSetField(final_phi, cfg.d_upper, cfg.d_lower),
                       metrics=report, loss_history=history, iters_run=res.iters, wall_time=wall,
                       loop_time=t_loop)
