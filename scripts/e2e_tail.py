"""Step timing of optimize()'s host side (dev probe): where the end-to-end
time goes beyond the device iterations."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, inputs, optimizer as op  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
cfg = b2.OptConfig(max_iters=K, stop_patience=10**9, precision="fp32")
b2.optimize(clip, focus, defocus, cfg)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = b2.optimize(clip, focus, defocus, cfg)
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t0
    T = [time.perf_counter()]
    target, m, fk, dk = op._prepare(clip, focus, defocus, cfg, None, None); T.append(time.perf_counter())
    td = nv.to_dev_staged(target, np.uint8); best = nv.empty(target.shape, np.float64)
    fmask = nv.empty(target.shape, np.uint8); hist = np.zeros((cfg.max_iters + 1, 7)); res = nv.LsopcResult()
    c = op._native_cfg(cfg); T.append(time.perf_counter())
    nv.check(nv.lib().lsopc_optimize(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c),
                                     nv.ptr(best), nv.ptr(fmask), hist.ctypes.data_as(ctypes.c_void_p),
                                     ctypes.byref(res), nv.stream()))
    T.append(time.perf_counter())
    sc = op._device_shots(fmask, nv.side_stream()); T.append(time.perf_counter())
    fm = nv.to_host(fmask); T.append(time.perf_counter())
    stage = nv.pinned_like(best); stage.copy_(best, non_blocking=True); torch.cuda.current_stream().synchronize()
    T.append(time.perf_counter())
    bp = np.empty(target.shape); np.copyto(bp, stage.numpy()); T.append(time.perf_counter())
    names = ["prepare", "upload+alloc", "lsopc_optimize", "device shots", "mask D2H", "phi D2H", "phi host copy"]
    print(f"optimize total {1e3 * t_all:.1f} ms ({K} iterations) | " +
          "  ".join(f"{n} {1e3 * (b - a):.2f}" for n, a, b in zip(names, T, T[1:])), flush=True)
