"""50 DSO iterations: CUDA-graph replay vs plain stream launches (dev probe;
run twice, with and without LSOPC_B200_NO_GRAPH=1)."""
import ctypes, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
fk = F.device(clip.shape); dk = D.device(clip.shape)
L = nv.lib(); sp = nv.stream(); td = nv.to_dev(clip, np.uint8)
c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=60, stop_patience=10**9))
for rep in range(3):
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c), sp, ctypes.byref(sess)))
    nv.check(L.lsopc_session_enqueue(sess, 5))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); nv.check(L.lsopc_session_enqueue(sess, 50)); e1.record(); torch.cuda.synchronize()
    print(f"{'stream' if os.environ.get('LSOPC_B200_NO_GRAPH') else 'graph '}: {e0.elapsed_time(e1)/50*1e3:.1f} us/iter")
    L.lsopc_session_destroy(sess)
