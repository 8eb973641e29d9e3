"""Time session create / iterations / finish separately (dev probe)."""
import sys, time, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
fk = focus.device(clip.shape); dk = defocus.device(clip.shape)
L = nv.lib(); sp = nv.stream()
td = nv.to_dev(clip, np.uint8)
c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=50, stop_patience=10**9))
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c), sp, ctypes.byref(sess)))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    nv.check(L.lsopc_session_enqueue(sess, 50)); torch.cuda.synchronize(); t2 = time.perf_counter()
    res = nv.LsopcResult(); hist = np.zeros((51, 7))
    nv.check(L.lsopc_session_finish(sess, None, None, hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res)))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    L.lsopc_session_destroy(sess); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  50 iters {1e3*(t2-t1):.1f} ms  finish {1e3*(t3-t2):.1f} ms  destroy {1e3*(t4-t3):.1f} ms")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = b2.optimize(clip, focus, defocus, b2.OptConfig(max_iters=50, stop_patience=10**9, precision="fp32"))
    torch.cuda.synchronize(); print(f"optimize: {1e3*(time.perf_counter()-t):.1f} ms")
