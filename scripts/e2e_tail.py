"""Step timing of optimize()'s host side (dev probe)."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs, optimizer as op
from paper_2303_12529_b200.metrics import shot_count
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
cfg = b2.OptConfig(max_iters=50, stop_patience=10**9, precision="fp32")
b2.optimize(clip, focus, defocus, cfg)
for rep in range(3):
    torch.cuda.synchronize(); T = [time.perf_counter()]
    target, m, fk, dk = op._prepare(clip, focus, defocus, cfg, None, None); T.append(time.perf_counter())
    td = nv.to_dev(target, np.uint8); best = nv.empty(target.shape, np.float64); fmask = nv.empty(target.shape, np.uint8)
    hist = np.zeros((cfg.max_iters + 1, 7)); res = nv.LsopcResult(); c = op._native_cfg(cfg); T.append(time.perf_counter())
    nv.check(nv.lib().lsopc_optimize(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c),
                                     nv.ptr(best), nv.ptr(fmask), hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res), nv.stream()))
    T.append(time.perf_counter())
    fm = nv.to_host(fmask); T.append(time.perf_counter())
    stage = nv.pinned_like(best); stage.copy_(best, non_blocking=True); torch.cuda.current_stream().synchronize(); T.append(time.perf_counter())
    bp = stage.numpy().copy(); T.append(time.perf_counter())
    sc = shot_count(fm); T.append(time.perf_counter())
    h = [op.IterationRecord(*(float(v) for v in row)) for row in hist[:res.iters]]; T.append(time.perf_counter())
    names = ["prepare", "alloc", "lsopc_optimize", "mask D2H", "phi D2H", "phi copy", "shot_count", "history"]
    print("  ".join(f"{n} {1e3*(b-a):.1f}" for n, a, b in zip(names, T, T[1:])), f"total {1e3*(T[-1]-T[0]):.1f} ms")
