#!/usr/bin/env python
"""Benchmark: DSO level-set ILT iterations/s on a 2048^2 clip, 24-kernel SOCS.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--precision fp32|fp64]

Workload (BASELINE.json configs[1]/[2]): synthetic ICCAD-2013-shaped metal
clip 2048 x 2048 @ 1 nm (`iccad_like_clip(seed=rank)`),
`gen_synthetic_kernels(35, 24, seed=4)` (24 focus + 24 defocus kernels),
OptConfig defaults, nominal + dose/defocus corners (L2 + PVB loss), curvature
on.  A "step" is one full DSO iteration (SOCS forward at 3 corners, losses,
best-iterate, adjoint, CG, level-set velocity, CFL and update) over one clip.
With N GPUs each rank optimises its own clip (clip-parallel, no collective):
`value` = total iterations/s over all ranks, timed with CUDA events, max over
ranks.  The stop rule is disabled for the timed steps (stop_patience = 1e9)
so every step does the full work.  Inputs are larger than L2 (24+24 spectra
= 768 MiB per iteration at FP32), so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_SIDE = 2048
K_SIDE, N_K, K_SEED = 35, 24, 4
METRIC = "ILT iters/s on 2048² clip (24-kernel SOCS); clips/s at 1/2/4/8 B200"


DATA = "synthetic (iccad_like_clip per rank, gen_synthetic_kernels(35,24,4))"


def workload_config(world):
    """The `config` of both arms (the precision tier is in `dtype`)."""
    return {"workload": "2048x2048 iccad_like_clip, SOCS 24+24 kernels K=35, 3 corners, one DSO iteration "
                        "per step (configs[1]); clip-parallel per GPU (configs[2])",
            "clip_side": N_SIDE, "kernels_per_set": N_K, "kernel_side": K_SIDE,
            "parallelism": f"clip-parallel x{world}",
            "l2_flush": "not needed: per-iteration working set (spectra 768 MiB+) > 126 MB L2"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-solve", action="store_true")
    p.add_argument("--no-tier", action="store_true", help="skip the other precision tier's sub-line")
    p.add_argument("--no-config0", action="store_true", help="skip the configs[0] 512^2 sub-line")
    p.add_argument("--clips", type=int, default=64, help="config 3 batch size (0 = skip)")
    p.add_argument("--tile", type=int, default=8192, help="config 5 tile side, split over the ranks (0 = skip)")
    p.add_argument("--tile-iters", type=int, default=6)
    p.add_argument("--dsn-batch", type=int, default=16, help="config 4 batch (0 = skip)")
    p.add_argument("--modsearch", type=int, default=41,
                   help="modulation_search candidates on one 2048^2 target, sharded over the ranks (0 = skip)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    """Roofline denominators: the driver's MEASURED_PEAKS.json (STREAM-style
    copy `hbm_gbs`), else the profiling guide's fallback."""
    try:
        pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        if float(pk.get("hbm_gbs", 0)) > 0:
            return pk, "measured"
    except Exception:
        pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def copy_rate_gbs(gib=2, reps=5):
    """Device-to-device copy rate of this GPU right now (read + write bytes),
    for context beside the roofline denominator."""
    import torch
    a = torch.empty(gib << 27, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del a, b
    return 2.0 * (gib << 30) / (ms * 1e6)


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (numpy/pocketfft, the reference's algorithm)


def cpu_iteration_sample(n_iters=1, threads=None, side=N_SIDE):
    from oracle import lsopc_oracle as o
    threads = threads or os.cpu_count() or 1
    o.use_threads(threads)
    try:
        clip = o.iccad_like_clip(0, n=side) if side == 2048 else o.two_bar_512()
        f, d = o.synthetic_kernels(K_SIDE, N_K, K_SEED)
        hf_f = o.spectra(f[0], clip.shape)
        hf_d = o.spectra(d[0], clip.shape)
        cfg = o.Cfg()
        phi = o.tsdf(clip)
        g_prev = d_prev = None
        times = []
        for it in range(n_iters):
            t0 = time.perf_counter()
            mask = o.mask_of(phi).astype(np.float64)
            prints, l_ilt, l_pvb, l_dso = o.forward_losses(mask, clip, f, d, cfg, hf_f, hf_d)
            g, dd, v, gm = o.step_fields(phi, mask, prints, None, clip, f, d, cfg, g_prev, d_prev,
                                         g_prev is None, hf_f, hf_d)
            dt, _ = o.cfl(v, cfg.eta)
            phi = np.clip(phi + dt * (-v * gm), cfg.d_lower, cfg.d_upper)
            g_prev, d_prev = g, dd
            times.append(time.perf_counter() - t0)
        return times, threads
    finally:
        o.use_threads(None)


# ---------------------------------------------------------------------------


def algorithmic_bytes_per_iter(n, n_k_total, prec):
    """FP32 tier n*(64 N_k + 170), FP64 tier n*(128 N_k + 230)
    with N_k kernels per set (n_k_total = 2 N_k)."""
    nk = n_k_total // 2
    return n * (64 * nk + 170) if prec == "fp32" else n * (128 * nk + 230)


PASS_NAMES = ["mask_fft (rows+cols)", "F1 forward cols: T_k = IFFT_y(M^.H_k)",
              "F2 forward rows: A_k = IFFT_x T_k, I = sum w|A_k|^2", "resist/loss/best",
              "A1 adjoint rows: U_k = FFT_x(gate.A_k)",
              "A2 adjoint cols: V = IFFT_y(sum w conj(H_k).FFT_y U_k)", "A3 finish: g = Re IFFT_x V (+CG dots)",
              "level-set step (velocity, CFL, update)"]


def pass_bytes(n, nk_tot, nsets, prec):
    """Algorithmic HBM bytes of each pass of one DSO iteration:
    c = complex element, r = real element of the transform tier."""
    c = 8 if prec == "fp32" else 16
    r = 4 if prec == "fp32" else 8
    per_px = [1 + 4 * c,                       # u8 mask in, M~ out+in, M^ out
              nk_tot * 2 * c + nsets * c,      # H_k in, T_k out; M^ tile once per (tile, set)
              nk_tot * 2 * c + nsets * r,      # T_k in, A_k out; I_set out
              4 * r + 1,                       # I_f, I_d in; gates out; target in
              nk_tot * 2 * c + nsets * r,      # A_k in, U_k out; gate once per (block, set)
              nk_tot * 2 * c + nsets * c,      # U_k in, H_k in; V_set out
              2 * c + 24,                      # V_f, V_d in; v out; v_prev in (dots)
              73]                              # phi stencil, v, d_prev, m in; d, u out; phi, mask out
    return [p * n for p in per_px]


def time_session(b2, nv, L, sp, focus, defocus, target, K, W, precision, world, dist, sampler=None):
    """W warm-up + K timed DSO iterations of one on-device session on
    `target` (stop rule disabled), CUDA events on the session stream, max over
    ranks.  Returns (ms over the K steps on this rank, max over ranks, the
    live session, launches per iteration)."""
    import contextlib
    import torch
    from paper_2303_12529_b200 import parallel
    shape = target.shape
    fk = focus.device(shape, precision)
    dk = defocus.device(shape, precision)
    cfg = b2.OptConfig(max_iters=W + K + 5, stop_patience=10**9, precision=precision)
    c = b2.optimizer._native_cfg(cfg)
    td = nv.to_dev(target, np.uint8)
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None,
                                    ctypes.byref(c), sp, ctypes.byref(sess)))
    nv.check(L.lsopc_session_enqueue(sess, W))
    stopped = ctypes.c_int()
    nv.check(L.lsopc_session_poll(sess, ctypes.byref(stopped), None))
    launches = L.lsopc_session_launches_per_iter(sess)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with (sampler if sampler is not None else contextlib.nullcontext()):
        ev0.record(stream)
        nv.check(L.lsopc_session_enqueue(sess, K))
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    nv.check(L.lsopc_session_poll(sess, ctypes.byref(stopped), None))
    assert not stopped.value, "stop rule fired inside the timed region"
    return ms, parallel.max_over_ranks(ms, device="cuda"), sess, launches


def time_e2e(b2, target, focus, defocus, K, precision, reps=3):
    """`b2.optimize` from a host uint8 target with K iterations (H2D, TSDF,
    K iterations, final prints, D2H of best phi + mask, device shot count): one
    warm-up call, then the median of `reps` (seconds)."""
    import torch
    cfg = b2.OptConfig(max_iters=K, stop_patience=10**9, precision=precision)
    b2.optimize(target, focus, defocus, cfg)
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = b2.optimize(target, focus, defocus, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        assert r.iters_run == K
    return statistics.median(times)


def time_solve(b2, target, warm_target, focus, defocus, precision):
    """Full default `optimize` to the reference's stop rule (configs[1]
    latency), after one warm-up solve on another target."""
    import torch
    b2.optimize(warm_target, focus, defocus, b2.OptConfig(precision=precision))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = b2.optimize(target, focus, defocus, b2.OptConfig(precision=precision))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, r


def b200_arm(args, world, rank, local):
    import torch
    import torch.distributed as dist

    # BENCH_DIST_BACKEND=gloo + BENCH_DEVICE=0 run several ranks on one GPU
    # (a functional check of the multi-rank paths; timings are then shared-GPU)
    dev = int(os.environ.get("BENCH_DEVICE", local))
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv
    from paper_2303_12529_b200 import inputs, parallel

    nv.set_precision(args.precision)
    K, W = args.steps, args.warmup
    clip = inputs.iccad_like_clip(seed=rank)
    (fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(K_SIDE, N_K, K_SEED)
    focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
    defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
    shape = clip.shape
    n = clip.size
    fk = focus.device(shape)
    dk = defocus.device(shape)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    L = nv.lib()

    # ---- device-resident timing: W warm-up + K timed iterations --------------
    clk = ClockSampler(dev)
    ms, ms_max, sess, launches_per_iter = time_session(b2, nv, L, sp, focus, defocus, clip, K, W, args.precision,
                                                       world, dist, clk)
    value = world * K / (ms_max / 1e3)

    # ---- per-pass CUDA-event timing on the session stream (after the timed region)
    pk, src = peaks()
    hbm = float(pk["hbm_gbs"])
    copy_gbs = copy_rate_gbs()
    ms_pass = (ctypes.c_double * 8)()
    nv.check(L.lsopc_session_time_passes(sess, 5, ms_pass))
    L.lsopc_session_destroy(sess)
    pb = pass_bytes(n, 2 * N_K, 2, args.precision)
    per_pass = {}
    for i in range(8):
        t = ms_pass[i] / 1e3
        per_pass[i] = {"name": PASS_NAMES[i], "us": t * 1e6, "bytes": pb[i],
                       "gbs": pb[i] / t / 1e9 if t > 0 else 0.0,
                       "frac": pb[i] / t / 1e9 / hbm if t > 0 else 0.0}
    dom = max(per_pass, key=lambda w: per_pass[w]["us"])
    iter_s = ms / 1e3 / K
    b_iter = algorithmic_bytes_per_iter(n, 2 * N_K, args.precision)
    traffic = dom_traffic = None
    tpath = ROOT / "profiles" / f"traffic_{args.precision}.json"
    if tpath.exists():
        try:
            tj = json.loads(tpath.read_text())
            traffic = tj.get("iteration")
            dom_traffic = tj.get(str(dom))
        except Exception:
            traffic = None

    # ---- e2e through the public API: host target in, host mask/phi out -------
    t_e2e = parallel.max_over_ranks(time_e2e(b2, clip, focus, defocus, K, args.precision), device="cuda")
    e2e_val = world * K / t_e2e

    def guard(fn):
        """A failed sub-line is reported in place and must not cost the
        headline line (one process; with several ranks an exception still
        propagates, since the other ranks' collectives would wait for it)."""
        if world > 1:
            return fn()
        try:
            return fn()
        except Exception as e:
            import traceback
            traceback.print_exc()
            try:
                torch.cuda.synchronize()
            except Exception:
                pass
            return {"error": f"{type(e).__name__}: {str(e)[:300]}"}

    # ---- config 2: full default solve of this rank's clip (latency) ----------
    def sec_solve():
        # warm-up solve on another clip: the first call with a new OptConfig
        # allocates the session buffers and captures the iteration graphs
        lat, rs = time_solve(b2, clip, inputs.iccad_like_clip(seed=1000 + rank), focus, defocus, args.precision)
        lat = parallel.max_over_ranks(lat, device="cuda")
        from paper_2303_12529_b200 import metrics as bm
        cfg_s = b2.OptConfig(precision=args.precision)
        nom = b2.print_corners(rs.final_mask, focus, defocus, cfg_s, binarize=True).nominal
        solve = {"iters": rs.iters_run, "latency_s": round(lat, 4), "wall_time_s": round(rs.wall_time, 4),
                 "l2": rs.metrics.l2, "pvband": rs.metrics.pvband, "shots": rs.metrics.shots,
                 "epe": bm.epe(nom, clip).as_dict(),
                 "note": "b2.optimize(iccad_like_clip(rank), OptConfig()) to the reference's stop rule; "
                         "incl. H2D, TSDF, final prints, D2H, shot count; after one warm-up solve"}
        # opt-in extensions (not in the reference), reported apart from the headline
        ext = {}
        for name, kw in (("upwind", {"grad_scheme": "upwind"}), ("reinit5", {"reinit_every": 5}),
                         ("upwind_reinit5", {"grad_scheme": "upwind", "reinit_every": 5})):
            cfg_x = b2.OptConfig(precision=args.precision, **kw)
            b2.optimize(inputs.iccad_like_clip(seed=1000 + rank), focus, defocus, cfg_x)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rx = b2.optimize(clip, focus, defocus, cfg_x)
            torch.cuda.synchronize()
            lx = time.perf_counter() - t0
            nx = b2.print_corners(rx.final_mask, focus, defocus, cfg_x, binarize=True).nominal
            ext[name] = {"iters": rx.iters_run, "latency_s": round(lx, 4), "l2": rx.metrics.l2,
                         "pvband": rx.metrics.pvband, "shots": rx.metrics.shots, "epe": bm.epe(nx, clip).as_dict(),
                         "best_l_dso": round(min(h.l_dso for h in rx.loss_history), 3)}
        solve["extensions"] = {"note": "opt-in OptConfig(grad_scheme='upwind') / reinit_every=5 (phi <- exact TSDF "
                                       "of its mask); not in the reference, parity against the oracle's "
                                       "restatement only", **ext}
        return solve

    # ---- config 3: a batch of clips sharded clip-parallel, no collective -----
    def sec_batch():
        # warm-up: every lane builds its spectra and session once
        parallel.warm_lanes(inputs.iccad_like_clip(seed=2000 + rank), focus, defocus,
                            b2.OptConfig(precision=args.precision))
        clips = parallel.LazyClips(args.clips, seed0=0)
        recs, secs = parallel.optimize_batch(clips, focus, defocus, b2.OptConfig(precision=args.precision),
                                             synchronize=torch.cuda.synchronize)
        batch = {"clips": args.clips, "seconds": round(secs, 3), "clips_per_s": round(args.clips / secs, 3),
                 "iters_total": int(sum(x.iters for x in recs)),
                 "iters_per_s": round(sum(x.iters for x in recs) / secs, 2),
                 "mean_l2": round(float(np.mean([x.l2 for x in recs])), 1),
                 "mean_pvband": round(float(np.mean([x.pvband for x in recs])), 1),
                 "note": f"iccad_like_clip(0..{args.clips - 1}) round-robin over {world} GPU(s), "
                         "2 concurrent streams per GPU, default OptConfig, each clip solved to the stop rule"}
        return batch

    solve = batch = None
    if not args.no_solve:
        solve = guard(sec_solve)
        if args.clips > 0:
            batch = guard(sec_batch)

    # ---- config 4: DevelSet-Net (random init) + GPU level-set refinement -----
    def sec_instant():
        from paper_2303_12529_b200 import dsn
        net = dsn.build_net()
        cfg_d = b2.OptConfig(precision=args.precision)
        dsn.instant_opc([inputs.iccad_like_clip(seed=900 + j) for j in range(2)], focus, defocus, cfg_d,
                        net=net)  # warm-up (both lanes)
        batch_t = [inputs.iccad_like_clip(seed=500 + rank * args.dsn_batch + i) for i in range(args.dsn_batch)]
        ri = dsn.instant_opc(batch_t, focus, defocus, cfg_d, net=net)
        lat = parallel.max_over_ranks(ri.latency, device="cuda")
        instant = {"batch": args.dsn_batch, "latency_s": round(lat, 4),
                   "stages_s": {"tsdf": round(ri.t_tsdf, 4), "dsn": round(ri.t_net, 4),
                                "init": round(ri.t_init, 4), "dso": round(ri.t_dso, 4)},
                   "iters_total": int(sum(x.iters_run for x in ri.results)),
                   "mean_l2": round(float(np.mean([x.metrics.l2 for x in ri.results])), 1),
                   "note": "random-init two-branch UNet (bf16) -> fused clip + AHF -> DSO per clip to the stop "
                           "rule (configs[3]); per rank"}
        return instant

    instant = None
    if args.dsn_batch > 0 and not args.no_solve:
        instant = guard(sec_instant)

    # ---- modulation_search, candidates sharded ---------
    def sec_modsearch():
        cfg_m = b2.OptConfig(precision=args.precision)
        tgt = inputs.iccad_like_clip(seed=0)
        phi_gt = b2.tsdf_from_mask(tgt)
        parallel.modulation_search_sharded(phi_gt, tgt, focus, defocus, cfg_m, num_samples=4,
                                           eval_steps=10, synchronize=torch.cuda.synchronize)  # warm-up
        rm, secs = parallel.modulation_search_sharded(phi_gt, tgt, focus, defocus, cfg_m,
                                                      num_samples=args.modsearch, eval_steps=10,
                                                      synchronize=torch.cuda.synchronize)
        modsearch = {"candidates": args.modsearch, "eval_steps": 10, "seconds": round(secs, 3),
                     "candidates_per_s": round(args.modsearch / secs, 2),
                     "best_delta_h": float(rm.best_delta_h),
                     "note": f"modulation_search(TSDF of iccad_like_clip(0), 41 shifts of the gate, 10 "
                             f"curvature-on iterations each, device-side final L_DSO); candidates round-robin "
                             f"over {world} GPU(s), 2 streams per GPU, one all-gather of the scores"}
        return modsearch

    modsearch = None
    if args.modsearch > 0 and not args.no_solve:
        modsearch = guard(sec_modsearch)

    # ---- config 5: one oversized tile split into strips over the ranks -------
    def sec_tile():
        from paper_2303_12529_b200 import tiled
        T = args.tile
        g = T // N_SIDE
        mosaic = inputs.mosaic_tile(range(g * g), grid=(g, g)) if g >= 1 and T % N_SIDE == 0 else \
            inputs.iccad_like_clip(seed=0, n=T)

        def run_tile(prec):
            cfg_t = b2.OptConfig(max_iters=args.tile_iters, stop_patience=10**9, precision=prec)
            tiled.optimize_tiled(mosaic, focus, defocus, b2.OptConfig(max_iters=1, stop_patience=10**9,
                                                                      precision=prec))  # warm-up
            rt = tiled.optimize_tiled(mosaic, focus, defocus, cfg_t)
            loop = parallel.max_over_ranks(rt.loop_time, device="cuda")
            hw = tuple(rt.window)
            kind = ("full-width row" if hw[0] < T else "full-height column" if hw[1] < T else "whole-tile")
            return {"side": T, "ranks": world, "strips": rt.strips, "window": list(rt.window),
                    "precision": prec, "iters": rt.iters_run, "loop_s": round(loop, 4),
                    "iters_per_s": round(rt.iters_run / loop, 3), "ms_per_iter": round(1e3 * loop / rt.iters_run, 2),
                    "note": f"{T}^2 mosaic of iccad_like_clips as {rt.strips} {kind} strip(s) "
                            f"({'x'.join(map(str, hw))} windows, {rt.strips // world} per rank) over "
                            f"{world} rank(s); 34-line phi halos, 3 combined scalar reductions per iteration "
                            "(configs[4])"}

        tile = run_tile(args.precision)
        if not args.no_tier:
            tile["tiers"] = {p: guard(lambda p=p: run_tile(p)) for p in ("fp32", "fp64") if p != args.precision}
        return tile

    tile = None
    if args.tile > 0 and not args.no_solve:
        tile = guard(sec_tile)

    # ---- the reference's own precision (fp64 tier: complex128 transforms) -----
    other = "fp64" if args.precision == "fp32" else "fp32"

    def sec_tiers():
        tiers = {}
        ms_o, ms_o_max, sess_o, _ = time_session(b2, nv, L, sp, focus, defocus, clip, K, W, other, world, dist)
        L.lsopc_session_destroy(sess_o)
        b_o = algorithmic_bytes_per_iter(n, 2 * N_K, other)
        t_o = parallel.max_over_ranks(time_e2e(b2, clip, focus, defocus, K, other), device="cuda")
        tiers[other] = {"value": round(world * K / (ms_o_max / 1e3), 3), "unit": "iters/s",
                        "ms_per_step": round(ms_o_max / K, 4),
                        "dtype": "c128 transforms / f64 level set" if other == "fp64" else
                                 "c64 transforms / f64 level set",
                        "e2e": {"value": round(world * K / t_o, 3), "unit": "iters/s"},
                        "roofline": {"bound": "hbm", "algorithmic_bytes": b_o,
                                     "achieved": round(b_o / (ms_o / 1e3 / K) / 1e9, 1), "peak": hbm,
                                     "frac": round(b_o / (ms_o / 1e3 / K) / 1e9 / hbm, 4)}}
        if not args.no_solve:
            lat_o, ro = time_solve(b2, clip, inputs.iccad_like_clip(seed=1000 + rank), focus, defocus, other)
            tiers[other]["solve"] = {"iters": ro.iters_run, "latency_s": round(parallel.max_over_ranks(
                lat_o, device="cuda"), 4), "l2": ro.metrics.l2, "pvband": ro.metrics.pvband,
                "shots": ro.metrics.shots}
        tiers[other]["note"] = (f"same workload as the headline in the {other} tier; device iters/s over {K} "
                                f"steps, e2e through b2.optimize, full default solve")
        return tiers

    tiers = guard(sec_tiers) if not args.no_tier else {}

    # ---- configs[0]: 512^2 two bars, 24 + 24 kernels, 50 iterations ---------
    def sec_config0():
        bars = inputs.two_bar_layout()
        c0 = {}
        for prec in (args.precision, other):
            ms0, ms0_max, s0, _ = time_session(b2, nv, L, sp, focus, defocus, bars, 50, W, prec, world, dist)
            L.lsopc_session_destroy(s0)
            t0e = parallel.max_over_ranks(time_e2e(b2, bars, focus, defocus, 50, prec), device="cuda")
            lat0, r0 = time_solve(b2, bars, inputs.rect_layout(512, [(100, 100, 80, 300)]), focus, defocus, prec)
            c0[prec] = {"iters_per_s": round(world * 50 / (ms0_max / 1e3), 2), "ms_per_iter": round(ms0_max / 50, 4),
                        "e2e_iters_per_s": round(world * 50 / t0e, 2),
                        "solve": {"iters": r0.iters_run, "latency_s": round(lat0, 4), "l2": r0.metrics.l2,
                                  "pvband": r0.metrics.pvband, "shots": r0.metrics.shots}}
        config0 = {"workload": "configs[0]: 512x512 two-bar target (test_acceptance.py:31), 24+24 kernels K=35, "
                               "OptConfig(max_iters=50, stop_patience=1e9) for iters/s (device: 50 graph-replayed "
                               "iterations; e2e: b2.optimize from the host target), plus the default solve "
                               "(reference: 17 iterations, l2 52, pvband 148, shots 102)", **c0}
        return config0

    config0 = None
    if not args.no_config0:
        config0 = guard(sec_config0)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        times, thr = cpu_iteration_sample(1)
        cpu = {"value": round(1.0 / times[0], 5), "unit": "iters/s", "cores": thr, "kind": "port",
               "sample": f"1 full DSO iteration of the numpy oracle (reference algorithm, pocketfft via "
                         f"scipy.fft on {thr} threads), iccad_like_clip(0) 2048^2, N_k=24, spectra "
                         f"and TSDF precomputed; {times[0]:.2f} s"}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "iters/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(ms_max / K, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c64 transforms / f64 level set" if args.precision == "fp32" else "c128 / f64",
        "data": DATA,
        "config": workload_config(world),
        "e2e": {"value": round(e2e_val, 3), "unit": "iters/s",
                "h2d_bytes_per_step": round(n / K), "d2h_bytes_per_step": round(9 * n / K),
                "note": f"b2.optimize(host uint8 target, max_iters={K}): H2D target, TSDF, {K} iterations, "
                        f"final prints, D2H best phi + mask, device shot count (lsopc_fracture_dev); median of 3 = {t_e2e:.3f} s"},
        # the roofline unit is one whole DSO iteration (one graph replay of
        # its launches): SURVEY §8(d) B_iter = n (64 N_k + 170) B (fp32 tier)
        # over the measured mean step time; the per-pass table beside it
        "roofline": {"bound": "hbm", "achieved": round(b_iter / iter_s / 1e9, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(b_iter / iter_s / 1e9 / hbm, 4), "traffic": traffic,
                     "kernel": f"one DSO iteration ({launches_per_iter} launches, CUDA graph)",
                     "algorithmic_bytes": b_iter,
                     "algorithmic_bytes_def": "SURVEY.md 8(d): n*(64*N_k + 170) (fp32), n*(128*N_k + 230) (fp64)",
                     "peak_source": src,
                     "copy_GBps_measured": round(copy_gbs, 1),
                     "frac_of_copy": round(b_iter / iter_s / 1e9 / copy_gbs, 4),
                     "dominant_pass": {"name": per_pass[dom]["name"], "us": round(per_pass[dom]["us"], 2),
                                       "pass_bytes": pb[dom], "GBps": round(per_pass[dom]["gbs"], 1),
                                       "frac": round(per_pass[dom]["frac"], 4), "traffic": dom_traffic},
                     "per_pass": {per_pass[w]["name"]: {"us": round(per_pass[w]["us"], 2),
                                                        "GBps": round(per_pass[w]["gbs"], 1),
                                                        "frac": round(per_pass[w]["frac"], 4)}
                                  for w in per_pass},
                     "iteration_passes": {"pass_bytes": sum(pb),
                                          "achieved_GBps_passes": round(sum(pb) / iter_s / 1e9, 1),
                                          "frac_passes": round(sum(pb) / iter_s / 1e9 / hbm, 4)}},
        "cpu_baseline": cpu,
        "gpu_launches": launches_per_iter * K,
        "clocks": clk.summary(),
        "solve": solve,
        "batch": batch,
        "tile": tile,
        "instant_opc": instant,
        "modulation_search": modsearch,
        "tiers": tiers,
        "config0": config0,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _ref_worker(idx, n_iters, barrier, q):
    """One single-threaded process of the reference arm: the numpy oracle
    (the reference algorithm on numpy's own pocketfft, which is single-threaded
    like the reference) -- untimed setup (spectra, TSDF), then `n_iters` timed
    DSO iterations on iccad_like_clip(idx) started together with the other
    processes."""
    try:
        sys.path.insert(0, str(ROOT))
        from oracle import lsopc_oracle as o
        clip = o.iccad_like_clip(idx)
        f, d = o.synthetic_kernels(K_SIDE, N_K, K_SEED)
        hf_f, hf_d = o.spectra(f[0], clip.shape), o.spectra(d[0], clip.shape)
        cfg = o.Cfg()
        phi = o.tsdf(clip)
        barrier.wait()
        t_start = time.time()
        g_prev = d_prev = None
        for it in range(n_iters):
            mask = o.mask_of(phi).astype(np.float64)
            prints, _, _, _ = o.forward_losses(mask, clip, f, d, cfg, hf_f, hf_d)
            g, dd, v, gm = o.step_fields(phi, mask, prints, None, clip, f, d, cfg, g_prev, d_prev,
                                         g_prev is None, hf_f, hf_d)
            dt, _ = o.cfl(v, cfg.eta)
            phi = np.clip(phi + dt * (-v * gm), cfg.d_lower, cfg.d_upper)
            g_prev, d_prev = g, dd
        q.put((idx, t_start, time.time(), None))
    except BaseException as e:  # report, never hang the parent
        try:
            barrier.abort()
        except Exception:
            pass
        q.put((idx, 0.0, 0.0, repr(e)))


def ref_processes(K):
    """P = min(cores, floor(0.8 RAM / 10 GB)) (one
    2048^2 oracle process peaks at ~9.8 GB), each running ceil(K / P)
    iterations so that at least K are timed."""
    cores = os.cpu_count() or 1
    try:
        import psutil
        ram = psutil.virtual_memory().total
    except Exception:
        ram = 64 << 30
    pmax = max(1, min(cores, int(0.8 * ram / (10 << 30))))
    pmax = int(os.environ.get("BENCH_REF_PROCS", pmax))
    p = max(1, min(pmax, K))
    return p, -(-K // p)


def reference_arm(args, world, rank):
    """The reference's CPU implementation of the path on this box's host
    cores: P concurrent single-threaded processes of the numpy oracle (the
    reference is single-threaded numpy; independent runs may execute
    concurrently), each on its own clip, started together after
    an untimed setup; value = all timed iterations / wall time from the first
    start to the last finish."""
    if rank != 0:
        return
    import multiprocessing as mp
    K = args.steps
    P, n_each = ref_processes(K)
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(P)
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(i, n_each, barrier, q)) for i in range(P)]
    for pr in procs:
        pr.start()
    res = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    errs = [r[3] for r in res if r[3]]
    if errs:
        raise RuntimeError(f"reference worker failed: {errs[0]}")
    wall = max(r[2] for r in res) - min(r[1] for r in res)
    total = P * n_each
    v = total / wall
    sample = (f"{P} concurrent single-threaded processes x {n_each} full DSO iteration(s) each of the numpy "
              f"oracle (reference algorithm, numpy pocketfft), iccad_like_clip(0..{P - 1}) 2048^2, N_k=24+24; "
              f"spectra + TSDF untimed; wall {wall:.1f} s")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "iters/s",
            "n_gpus": world, "steps": total, "warmup": 0, "ms_per_step": round(1e3 / v, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 / f64",
            "data": DATA, "config": workload_config(world),
            "cpu_baseline": {"value": round(v, 5), "unit": "iters/s", "cores": P, "kind": "port",
                             "sample": sample},
            "clips_per_s_derived": round(v / 25.0, 6),
            "clips_note": "configs[2] CPU clips/s = iters/s / 25 (the configs[1] solve takes 25 iterations)",
            "e2e": {"value": round(v, 5), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, world, rank)
    else:
        b200_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
