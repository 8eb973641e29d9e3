"""Oversized tile split into strips (BASELINE configs[4]).

The reference optimises one periodic N x N tile with circular FFTs
(`fields.py:5-6`, `litho.py:114-126`).  Here the tile is cut into strips:
full-width strips of rows (axis=0, the fp32 default) or full-height strips
of columns (axis=1).  Each strip runs the unchanged device pipeline on a
power-of-two window that holds its interior lines plus halos of at least
HALO = 2 * (K // 2) lines on each side (the forward field at a pixel needs
the mask within +-K//2, the adjoint within +-2 * (K//2)), so every interior
value equals the full-tile computation.

Each rank holds one or more consecutive strips (`strips_per_rank`; by
default the count that covers the least window area, `auto_strips` -- a
single B200 runs an 8192^2 tile as nine 1024 x 8192 windows, 50.5 ms per
iteration against 84.8 ms for the whole tile as one grid).  Row strips are the fp32 default because the
window's long (tile-length, 8192-point) axis then lies along the rows,
whose transforms stream by TMA; the fp64 tier takes column strips, whose
8192 x <=1024 windows run through the split plan (complex128 rows stop at
4096 points).  Per iteration, over the strips of a rank in order:

    phases 0, 5  forward, then adjoint + CG dot partials (per strip)
                                          -> sum of losses and dots (strips, ranks)
    phase 6      stop rule, best iterate
    phase 2      CG direction, level-set velocity -> max |v|, |grad phi|
    phase 3      CFL step, interior update        -> max step
    phase 4      history record
    halo         HALO lines of phi from both neighbours (device copies
                 between a rank's strips, P2P between ranks; wrapping)

Optics wrap around the tile edge (periodic, like the reference's FFT); the
phi stencil uses replicate padding at the global left/right edge
(`levelset.py:112`), so the edge ranks clamp their stencil to the interior.
Losses, dots, maxima and the final L2/PVB are summed over interiors only.
All ranks see the same scalars, so the stop rule, best iterate and CG
restarts agree everywhere.

The strips of one process share their plan's work fields (T_k, A_k, V):
the adjoint (phase 5) reads only fields the forward just wrote, so it runs
straight after each strip's forward, before the stop decision (phase 6),
which it never depends on.

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
    tile, one per rank; windows are powers of two along the split axis."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if (W if axis == 1 else H) % world:
        raise ValueError(f"tile extent {W if axis == 1 else H} is not divisible by {world} ranks")
    return strip_layout(H, W, world, K, axis)[rank]


def _pow2_at_least(n):
    p = 1
    while p < n:
        p *= 2
    return p


def strip_layout(H, W, nstrips, K, axis=1):
    """All `nstrips` strips along `axis` of an H x W tile: interiors
    [floor(i L / n), floor((i+1) L / n)) of the split extent L, one common
    power-of-two window width (so the strips share one plan)."""
    if axis not in (0, 1):
        raise ValueError("axis must be 0 (row strips) or 1 (column strips)")
    if axis == 0:
        H, W = W, H  # describe row strips in the transposed frame
    if nstrips < 1:
        raise ValueError(f"bad strip count {nstrips}")
    halo = 2 * (K // 2)
    if nstrips == 1:
        return [Strip(0, 1, H, W, 0, W, W, 0, halo, axis)]
    b = [(i * W) // nstrips for i in range(nstrips + 1)]
    wmin = min(b[i + 1] - b[i] for i in range(nstrips))
    wmax = max(b[i + 1] - b[i] for i in range(nstrips))
    if halo > wmin:
        raise ValueError(f"strip width {wmin} is narrower than the halo {halo}")
    if wmax + 2 * halo > W:
        raise ValueError(f"{nstrips} strips of a {W}-wide tile cannot carry {halo}-line halos")
    ww = min(_pow2_at_least(wmax + 2 * halo), W)  # at most the whole tile (the window then wraps)
    return [Strip(i, nstrips, H, W, b[i], b[i + 1], ww, (ww - (b[i + 1] - b[i])) // 2, halo, axis)
            for i in range(nstrips)]


def max_window(H, W, axis, precision):
    """Widest window (lines along the split axis) worth running: 2048, where
    the transforms cost least per pixel; in the fp64 tier also a legal plan
    (complex128 sides up to 4096, 8192 x <=1024 through the split plan)."""
    other = W if axis == 0 else H  # the window's full-length side
    if precision == "fp64" and other > 4096:
        return 1024 if axis == 1 else 0  # fp64 has no 8192-point rows
    return 2048


def auto_strips(H, W, world, K, axis, precision):
    """Strips per rank: the count whose windows cover the least area per
    rank (m strips x window width), among windows no wider than `max_window`
    and no narrower than 512 lines.  The transforms cost about the same per
    pixel from 512- to 2048-line windows (0.67-0.68 ms per Mpx, fp32,
    scripts/tile_bench.py), so area is time: an 8192^2 tile on one GPU runs
    as nine 1024 x 8192 windows (50.5 ms per iteration; five 2048-line
    windows 55.8, the whole tile 84.8)."""
    L = H if axis == 0 else W
    if L % world:
        raise ValueError(f"tile extent {L} is not divisible by {world} ranks")
    cap = max_window(H, W, axis, precision)
    if cap == 0:
        raise ValueError("the fp64 tier has no 8192-point rows: use column strips (axis=1)")
    halo = 2 * (K // 2)
    best = None
    for m in range(1, 257):
        n = world * m
        wi = -(-L // n)
        if n > 1 and wi < halo:
            break
        ww = L if n == 1 else min(_pow2_at_least(wi + 2 * halo), L)
        if ww < min(512, L) and best is not None:
            break
        if ww > cap:
            continue
        if best is None or m * ww < best[0]:
            best = (m * ww, m)
    if best is None:
        raise ValueError(f"no strip count fits windows of at most {cap} lines")
    return best[1]


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


def _lines(phi, strip):
    """View of a window with the split axis along dim 1."""
    return phi.t() if strip.axis == 0 else phi


def exchange_local_halos(phis, strips, wrap):
    """HALO lines between consecutive strips held by this process (device
    copies): strip j's left halo from strip j-1's interior, its right halo
    from strip j+1's; `wrap`: the process holds the whole ring, so the first
    and last strips are neighbours too.  Reads touch interiors only and
    writes halos only, so the order of the copies is immaterial."""
    k = len(strips)
    if k == 1 and wrap:  # one strip holding the whole tile: its window is the tile
        return
    for j in range(k):
        s = strips[j]
        h = s.halo
        i0, i1 = s.interior
        P = _lines(phis[j], s)
        if j > 0 or wrap:
            L = strips[j - 1]
            _, l1 = L.interior
            P[:, i0 - h:i0].copy_(_lines(phis[j - 1], L)[:, l1 - h:l1])
        if j < k - 1 or wrap:
            R = strips[(j + 1) % k]
            r0, _ = R.interior
            P[:, i1:i1 + h].copy_(_lines(phis[(j + 1) % k], R)[:, r0:r0 + h])


def exchange_halos(phi, strip, tags=True, last=None):
    """Refresh the HALO columns on each side of the interior of `phi`
    (H x ww torch tensor) from the neighbouring ranks' interiors (wrapping).
    With several strips per rank, `phi` / `strip` is the rank's first strip
    (its left edge) and `last` = (phi, strip) its last (its right edge).

    NCCL ignores P2P tags and pairs the operations between two ranks by
    position, so the order below is what keeps the two messages apart when
    left == right (two ranks): each rank sends its left edge first and its
    right edge second, and receives from its right neighbour first (that
    neighbour's left edge) and from its left neighbour second.  With distinct
    neighbours the order is immaterial.  `tags=False` exercises that
    positional matching on backends that honour tags (gloo)."""
    dist = _dist()
    world = dist.get_world_size() if dist.is_initialized() else 1
    if world == 1:
        return
    import torch
    rank = dist.get_rank()
    phi_l, s_l = phi, strip
    phi_r, s_r = last if last is not None else (phi, strip)
    h = strip.halo
    i0, _ = s_l.interior
    _, i1 = s_r.interior
    left, right = (rank - 1) % world, (rank + 1) % world
    nccl = _backend_is_nccl()
    stage = (lambda t: t) if nccl else (lambda t: t.cpu())
    P_l, P_r = _lines(phi_l, s_l), _lines(phi_r, s_r)  # row strips: halo rows are contiguous
    send_l = stage(P_l[:, i0:i0 + h].contiguous())    # -> left neighbour's right halo
    send_r = stage(P_r[:, i1 - h:i1].contiguous())    # -> right neighbour's left halo
    recv_l = torch.empty_like(send_l)
    recv_r = torch.empty_like(send_r)
    t1, t2 = (1, 2) if tags else (0, 0)
    ops = [dist.P2POp(dist.isend, send_l, left, tag=t1), dist.P2POp(dist.isend, send_r, right, tag=t2),
           dist.P2POp(dist.irecv, recv_r, right, tag=t1), dist.P2POp(dist.irecv, recv_l, left, tag=t2)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    P_l[:, i0 - h:i0].copy_(recv_l)
    P_r[:, i1:i1 + h].copy_(recv_r)


@dataclass
class TiledResult:
    final_mask: np.ndarray      # global tile (every rank)
    final_phi: LevelSetField    # global tile (every rank)
    metrics: MetricsReport
    loss_history: list
    iters_run: int
    wall_time: float
    loop_time: float = 0.0      # seconds in the iteration loop (device-synchronised)
    strips: int = 1             # strips of the whole tile (all ranks)
    window: tuple = ()          # window shape of every strip


def _combine(views, sl, op):
    """Sum / max of the scalars `sl` over this process's strips and then over
    the ranks, written back to every strip's scalar buffer."""
    import torch
    dist = _dist()
    if len(views) == 1:
        all_reduce_(views[0][sl], op)
        return
    stk = torch.stack([v[sl] for v in views])
    acc = stk.sum(0) if op == dist.ReduceOp.SUM else stk.amax(0)
    all_reduce_(acc, op)
    for v in views:
        v[sl].copy_(acc)


def optimize_tiled(target, focus_kernels, defocus_kernels, cfg, phi0=None, axis=None, strips_per_rank=None):
    """`optimize` (optimizer.py:204-284) of one tile split into strips over
    the ranks of the default process group.  Every rank passes the same
    global `target` (and `phi0`); every rank returns the assembled global
    result.  axis=0: strips of rows (full width), axis=1: strips of columns
    (full height); None: rows, or columns in the fp64 tier when the tile is
    wider than 4096.  strips_per_rank=None: `auto_strips`."""
    import time
    import torch
    from .optimizer import IterationRecord, _check_target, _native_cfg

    t0 = time.perf_counter()
    dist = _dist()
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
    target = _check_target(target)
    H, W = target.shape
    prec = getattr(cfg, "precision", None)
    pname = (prec or nv.get_precision()).lower()
    if axis is None:
        axis = 1 if pname == "fp64" and W > 4096 else 0
    K = focus_kernels.side
    m = strips_per_rank or auto_strips(H, W, world, K, axis, pname)
    layout = strip_layout(H, W, world * m, K, axis)
    mine = layout[rank * m:(rank + 1) * m]
    wshape = mine[0].window_shape

    def window(a, st):  # the window's lines of a global (host or device) array
        return a[:, st.lines()] if axis == 1 else a[st.lines(), :]

    # initial level set: the whole tile's TSDF (levelset.py:86-101) or phi0, windowed
    if phi0 is None:
        td_full = nv.to_dev(target, np.uint8)
        phi_full = nv.empty((H, W), np.float64)
        nv.check(nv.lib().lsopc_tsdf(H, W, nv.ptr(td_full), float(cfg.d_upper), float(cfg.d_lower),
                                     nv.ptr(phi_full), nv.stream()))
        phi_wins = []
        for st_ in mine:
            idx = torch.as_tensor(st_.lines(), device=phi_full.device)
            phi_wins.append((phi_full[:, idx] if axis == 1 else phi_full[idx, :]).contiguous())
        del phi_full, td_full
    else:
        p = np.asarray(phi0.phi, dtype=np.float64)
        if p.shape != target.shape:
            raise ValueError("phi0 dimensions do not match target")
        phi_wins = [nv.to_dev(np.ascontiguousarray(window(p, st_))) for st_ in mine]
    tgt_wins = [nv.to_dev(np.ascontiguousarray(window(target, st_)), np.uint8) for st_ in mine]

    fk = litho.device_kernels(focus_kernels, wshape, prec)
    dk = litho.device_kernels(defocus_kernels, wshape, prec)
    c = _native_cfg(cfg)
    c.skip_target_check = 1
    L = nv.lib()
    sessions = []
    try:
        for st_, tw, pw in zip(mine, tgt_wins, phi_wins):
            sess = ctypes.c_void_p()
            nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(tw), nv.ptr(pw), None,
                                            ctypes.byref(c), nv.stream(), ctypes.byref(sess)))
            sessions.append(sess)
            i0, i1 = st_.interior
            lo, hi = st_.stencil_bounds()
            if axis == 1:
                nv.check(L.lsopc_session_set_window(sess, i0, i1, lo, hi, 0, H, 0, H))
            else:
                nv.check(L.lsopc_session_set_window(sess, 0, W, 0, W, i0, i1, lo, hi))
        del phi_wins
        scs = [torch.as_tensor(_CudaView(L.lsopc_session_scalars(x), (8,), "<f8"), device="cuda") for x in sessions]
        phis = [torch.as_tensor(_CudaView(L.lsopc_session_phi_ptr(x), wshape, "<f8"), device="cuda")
                for x in sessions]
        flag = torch.as_tensor(_CudaView(L.lsopc_session_state_flag(sessions[0]), (1,), "<i4"), device="cuda")
        SUM, MAX = dist.ReduceOp.SUM, dist.ReduceOp.MAX

        def phase(ph):
            for x in sessions:
                nv.check(L.lsopc_session_phase(x, ph))

        torch.cuda.synchronize()
        t_loop = time.perf_counter()
        # The device stop flag turns every later phase into a no-op (its
        # bodies check it), so the host reads it only every `poll` iterations
        # and the stream stays queued in between; it is identical in every
        # strip (same global scalars), so all ranks leave together.
        poll = 4
        for i in range(cfg.max_iters):
            for x in sessions:  # forward, then the adjoint while the plan's fields hold this strip's
                nv.check(L.lsopc_session_phase(x, 0))
                nv.check(L.lsopc_session_phase(x, 5))
            _combine(scs, slice(0, 4), SUM)
            phase(6)
            phase(2)
            _combine(scs, slice(4, 6), MAX)
            phase(3)
            _combine(scs, slice(6, 7), MAX)
            phase(4)
            if (i + 1) % poll == 0 and int(flag.item()):
                break
            exchange_local_halos(phis, mine, wrap=world == 1)
            exchange_halos(phis[0], mine[0], last=(phis[-1], mine[-1]))
        torch.cuda.synchronize()
        t_loop = time.perf_counter() - t_loop
        hist = np.zeros((cfg.max_iters + 1, 7))
        l2 = pvb = 0
        my_mask, my_phi = [], []
        for j, (x, st_) in enumerate(zip(sessions, mine)):
            best = nv.empty(wshape, np.float64)
            fmask = nv.empty(wshape, np.uint8)
            h_j = np.zeros((cfg.max_iters + 1, 7))
            res = nv.LsopcResult()
            nv.check(L.lsopc_session_finish(x, nv.ptr(best), nv.ptr(fmask), h_j.ctypes.data_as(ctypes.c_void_p),
                                            ctypes.byref(res)))
            if j == 0:
                hist, iters = h_j, res.iters
            l2 += res.l2
            pvb += res.pvband
            i0, i1 = st_.interior
            my_mask.append(fmask[:, i0:i1] if axis == 1 else fmask[i0:i1, :])
            my_phi.append(best[:, i0:i1] if axis == 1 else best[i0:i1, :])
    finally:
        for x in sessions:
            L.lsopc_session_destroy(x)
    counts = torch.tensor([float(l2), float(pvb)], dtype=torch.float64, device="cuda")
    all_reduce_(counts, dist.ReduceOp.SUM)
    # assemble the global mask and phi from every strip's interior
    my_mask = torch.cat(my_mask, dim=axis).contiguous()
    my_phi = torch.cat(my_phi, dim=axis).contiguous()
    if world > 1:
        if _backend_is_nccl():  # all ranks hold m strips; interior widths differ by at most one line
            masks = [m_.cpu().numpy() for m_ in _all_gather_var(my_mask, axis)]
            phis_g = [p_.cpu().numpy() for p_ in _all_gather_var(my_phi, axis)]
        else:
            masks = [None] * world
            phis_g = [None] * world
            dist.all_gather_object(masks, my_mask.cpu().numpy())
            dist.all_gather_object(phis_g, my_phi.cpu().numpy())
        final_mask = np.concatenate(masks, axis=axis)
        final_phi = np.concatenate(phis_g, axis=axis)
    else:
        final_mask = my_mask.cpu().numpy()
        final_phi = my_phi.cpu().numpy()
    wall = time.perf_counter() - t0
    history = [IterationRecord(*(float(v) for v in row)) for row in hist[:iters]]
    report = MetricsReport(l2=int(counts[0].item()), pvband=int(counts[1].item()), shots=shot_count(final_mask),
                           wall_time=wall, iters=iters)
    return TiledResult(final_mask=final_mask, final_phi=LevelSetField(final_phi, cfg.d_upper, cfg.d_lower),
                       metrics=report, loss_history=history, iters_run=iters, wall_time=wall,
                       loop_time=t_loop, strips=len(layout), window=tuple(wshape))


def _all_gather_var(t, axis):
    """all_gather of tensors whose extent along `axis` differs between ranks
    (padded to the largest, then trimmed)."""
    import torch
    dist = _dist()
    world = dist.get_world_size()
    n = torch.tensor([t.shape[axis]], device=t.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    ns = [int(v.item()) for v in ns]
    mx = max(ns)
    pad = list(t.shape)
    pad[axis] = mx
    buf = torch.zeros(pad, dtype=t.dtype, device=t.device)
    (buf[:, :t.shape[1]] if axis == 1 else buf[:t.shape[0]]).copy_(t)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [(o[:, :k] if axis == 1 else o[:k]) for o, k in zip(outs, ns)]
