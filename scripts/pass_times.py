"""Per-pass CUDA-event times of the DSO iteration (dev probe; works with the
experiment builds selected by LSOPC_B200_LIB)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
side = int(sys.argv[2]) if len(sys.argv) > 2 else 2048       # 8192: configs[4] mosaic tile
width = int(sys.argv[3]) if len(sys.argv) > 3 else side       # < side: a strip window
nv.set_precision(prec)
if side == 2048:
    clip = inputs.iccad_like_clip(seed=0)
else:
    g = side // 2048
    clip = np.ascontiguousarray(inputs.mosaic_tile(range(g * g), grid=(g, g))[:, :width])
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
fk = focus.device(clip.shape); dk = defocus.device(clip.shape)
L = nv.lib(); sp = nv.stream()
td = nv.to_dev(clip, np.uint8)
c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=40, stop_patience=10**9))
sess = ctypes.c_void_p()
nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c), sp, ctypes.byref(sess)))
ms = (ctypes.c_double * 8)()
nv.check(L.lsopc_session_time_passes(sess, 3, ms))
nv.check(L.lsopc_session_time_passes(sess, 10, ms))
names = ["mask", "F1", "F2", "resist", "A1", "A2", "A3", "ls"]
print(f"{prec} {clip.shape[0]}x{clip.shape[1]}:", " ".join(f"{n}={ms[i]*1e3:.0f}us" for i, n in enumerate(names)),
      f"total={sum(ms)*1e3:.0f}us")
