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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-solve", action="store_true")
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
    cfg = b2.OptConfig(max_iters=W + K + 5, stop_patience=10**9, precision=args.precision)
    c = b2.optimizer._native_cfg(cfg)
    td = nv.to_dev(clip, np.uint8)
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None,
                                    ctypes.byref(c), sp, ctypes.byref(sess)))
    nv.check(L.lsopc_session_enqueue(sess, W))
    stopped = ctypes.c_int()
    nv.check(L.lsopc_session_poll(sess, ctypes.byref(stopped), None))
    launches_per_iter = L.lsopc_session_launches_per_iter(sess)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        nv.check(L.lsopc_session_enqueue(sess, K))
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    nv.check(L.lsopc_session_poll(sess, ctypes.byref(stopped), None))
    assert not stopped.value, "stop rule fired inside the timed region"
    ms_max = parallel.max_over_ranks(ms, device="cuda")
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
    traffic = None
    tpath = ROOT / "profiles" / f"traffic_{args.precision}.json"
    if tpath.exists():
        try:
            traffic = json.loads(tpath.read_text()).get(str(dom))
        except Exception:
            traffic = None

    # ---- e2e through the public API: host target in, host mask/phi out -------
    # b2.optimize(host uint8 target) with K iterations: H2D of the target,
    # TSDF, K iterations, final hard prints, D2H of best phi + final mask, and
    # the host shot count, all inside the timed call.  One warm-up call, then
    # the median of 3 (max over ranks).
    cfg_e2e = b2.OptConfig(max_iters=K, stop_patience=10**9, precision=args.precision)
    b2.optimize(clip, focus, defocus, cfg_e2e)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = b2.optimize(clip, focus, defocus, cfg_e2e)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        assert r.iters_run == K
    t_e2e = parallel.max_over_ranks(statistics.median(times), device="cuda")
    e2e_val = world * K / t_e2e

    # ---- config 2: full default solve of this rank's clip (latency) ----------
    solve = batch = None
    if not args.no_solve:
        # warm-up solve on another clip: the first call with a new OptConfig
        # allocates the session buffers and captures the iteration graphs
        b2.optimize(inputs.iccad_like_clip(seed=1000 + rank), focus, defocus, b2.OptConfig(precision=args.precision))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = b2.optimize(clip, focus, defocus, b2.OptConfig(precision=args.precision))
        torch.cuda.synchronize()
        lat = parallel.max_over_ranks(time.perf_counter() - t0, device="cuda")
        solve = {"iters": rs.iters_run, "latency_s": round(lat, 4), "wall_time_s": round(rs.wall_time, 4),
                 "l2": rs.metrics.l2, "pvband": rs.metrics.pvband, "shots": rs.metrics.shots,
                 "note": "b2.optimize(iccad_like_clip(rank), OptConfig()) to the reference's stop rule; "
                         "incl. H2D, TSDF, final prints, D2H, shot count; after one warm-up solve"}
        # ---- config 3: a batch of clips sharded clip-parallel, no collective ---
        if args.clips > 0:
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

    # ---- config 4: DevelSet-Net (random init) + GPU level-set refinement -----
    instant = None
    if args.dsn_batch > 0 and not args.no_solve:
        from paper_2303_12529_b200 import dsn
        net = dsn.build_net()
        cfg_d = b2.OptConfig(precision=args.precision)
        dsn.instant_opc([inputs.iccad_like_clip(seed=900)], focus, defocus, cfg_d, net=net)  # warm-up
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

    # ---- modulation_search, candidates sharded ---------
    modsearch = None
    if args.modsearch > 0 and not args.no_solve:
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

    # ---- config 5: one oversized tile split into strips over the ranks -------
    tile = None
    if args.tile > 0 and not args.no_solve:
        from paper_2303_12529_b200 import tiled
        T = args.tile
        g = T // N_SIDE
        mosaic = inputs.mosaic_tile(range(g * g), grid=(g, g)) if g >= 1 and T % N_SIDE == 0 else \
            inputs.iccad_like_clip(seed=0, n=T)
        cfg_t = b2.OptConfig(max_iters=args.tile_iters, stop_patience=10**9, precision=args.precision)
        tiled.optimize_tiled(mosaic, focus, defocus, b2.OptConfig(max_iters=1, stop_patience=10**9,
                                                                  precision=args.precision))  # warm-up
        rt = tiled.optimize_tiled(mosaic, focus, defocus, cfg_t)
        loop = parallel.max_over_ranks(rt.loop_time, device="cuda")
        st = tiled.strip_geometry(T, T, world, rank, K_SIDE)
        tile = {"side": T, "ranks": world, "window": [T, st.ww], "iters": rt.iters_run,
                "loop_s": round(loop, 4), "iters_per_s": round(rt.iters_run / loop, 3),
                "ms_per_iter": round(1e3 * loop / rt.iters_run, 2),
                "note": f"{T}^2 mosaic of iccad_like_clips, full-height strips over {world} rank(s), "
                        "34-column phi halo exchange + 4 scalar all-reduces per iteration (configs[4])"}

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
        "data": "synthetic (iccad_like_clip per rank, gen_synthetic_kernels(35,24,4))",
        "config": {"workload": "2048x2048 iccad_like_clip, SOCS 24+24 kernels K=35, 3 corners, "
                               "one DSO iteration per step (configs[1]); clip-parallel per GPU (configs[2])",
                   "clip_side": N_SIDE, "kernels_per_set": N_K, "kernel_side": K_SIDE,
                   "precision_tier": args.precision, "parallelism": f"clip-parallel x{world}",
                   "l2_flush": "not needed: per-iteration working set (spectra 768 MiB+) > 126 MB L2"},
        "e2e": {"value": round(e2e_val, 3), "unit": "iters/s",
                "h2d_bytes_per_step": round(n / K), "d2h_bytes_per_step": round(9 * n / K),
                "note": f"b2.optimize(host uint8 target, max_iters={K}): H2D target, TSDF, {K} iterations, "
                        f"final prints, D2H best phi + mask, host shot count; median of 3 = {t_e2e:.3f} s"},
        "roofline": {"bound": "hbm", "achieved": round(per_pass[dom]["gbs"], 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(per_pass[dom]["frac"], 4), "traffic": traffic,
                     "kernel": per_pass[dom]["name"], "peak_source": src,
                     "copy_GBps_measured": round(copy_gbs, 1),
                     "frac_of_copy": round(per_pass[dom]["gbs"] / copy_gbs, 4),
                     "per_pass": {per_pass[w]["name"]: {"us": round(per_pass[w]["us"], 2),
                                                        "GBps": round(per_pass[w]["gbs"], 1),
                                                        "frac": round(per_pass[w]["frac"], 4)}
                                  for w in per_pass},
                     "iteration": {"algorithmic_bytes_survey": b_iter,
                                   "achieved_GBps_survey": round(b_iter / iter_s / 1e9, 1),
                                   "frac_survey": round(b_iter / iter_s / 1e9 / hbm, 4),
                                   "pass_bytes": sum(pb),
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
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, world, rank):
    if rank != 0:
        return
    K = args.steps
    budget_s = float(os.environ.get("BENCH_REF_BUDGET_S", "150"))
    times, thr = cpu_iteration_sample(1)
    n_more = max(0, min(K, int(budget_s / max(times[0], 1e-3))) - 1)
    if n_more:
        t2, _ = cpu_iteration_sample(n_more + 1)
        times = t2
    v = len(times) / sum(times)
    sample = (f"{len(times)} full DSO iteration(s) of the numpy oracle port (reference algorithm, "
              f"pocketfft via scipy.fft on {thr} threads), iccad_like_clip(0) 2048^2, N_k=24; "
              f"requested steps={K}, bounded to ~{budget_s:.0f} s")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "iters/s",
            "n_gpus": world, "steps": len(times), "warmup": 0, "ms_per_step": round(1e3 / v, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 / f64",
            "data": "synthetic", "config": {"workload": "2048x2048 iccad_like_clip, SOCS 24+24, one DSO iteration"},
            "cpu_baseline": {"value": round(v, 5), "unit": "iters/s", "cores": thr, "kind": "port",
                             "sample": sample},
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
