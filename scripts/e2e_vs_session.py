"""Per-iteration device time: a session's enqueue(K) (bench value) against
lsopc_optimize (the e2e path), same process and box (dev probe)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, inputs  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
nv.set_precision(prec)
L = nv.lib()
clip = inputs.iccad_like_clip(seed=0)
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
fk, dk = focus.device(clip.shape, prec), defocus.device(clip.shape, prec)
td = nv.to_dev(clip, np.uint8)
s = torch.cuda.current_stream()


def ev_time(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for K in (20, 40):
    c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=K + 10, stop_patience=10**9, precision=prec))
    sess = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c),
                                    nv.stream(), ctypes.byref(sess)))
    nv.check(L.lsopc_session_enqueue(sess, 5))
    ms_s = ev_time(lambda: nv.check(L.lsopc_session_enqueue(sess, K)))
    L.lsopc_session_destroy(sess)
    c2 = b2.optimizer._native_cfg(b2.OptConfig(max_iters=K, stop_patience=10**9, precision=prec))
    best, fm = nv.empty(clip.shape, np.float64), nv.empty(clip.shape, np.uint8)
    hist = np.zeros((K + 1, 7))
    res = nv.LsopcResult()
    run = lambda: nv.check(L.lsopc_optimize(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None,  # noqa: E731
                                            ctypes.byref(c2), nv.ptr(best), nv.ptr(fm),
                                            hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(res), nv.stream()))
    run()
    ms_o = min(ev_time(run) for _ in range(3))
    print(f"{prec} K={K}: session enqueue {ms_s / K:.3f} ms/iter; lsopc_optimize {ms_o:.2f} ms total "
          f"({ms_o / K:.3f} ms/iter incl. setup)", flush=True)
