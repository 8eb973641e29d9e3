"""Per-pass CUDA-event times (lsopc_session_time_passes) of one DSO iteration
on tall / wide / square grids, 24 + 24 kernels (configs[4] geometry
study).  [PREC=fp64] python scripts/tile_passes.py H W [H W ...]"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, inputs  # noqa: E402

NAMES = ["mask", "F1", "F2", "resist", "A1", "A2", "A3", "ls"]
nv.set_precision(os.environ.get("PREC", "fp32"))
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
args = [int(a) for a in sys.argv[1:]] or [8192, 2048, 2048, 8192]
for H, W in zip(args[::2], args[1::2]):
    big = inputs.mosaic_tile(range(16), grid=(4, 4))
    # small grids: the centre of the first clip (its wires lie in [512, 1536)^2)
    y0 = 1024 - H // 2 if H <= 2048 else 0
    x0 = 1024 - W // 2 if W <= 2048 else 0
    t = np.ascontiguousarray(big[y0:y0 + H, x0:x0 + W])
    fk, dk = focus.device((H, W)), defocus.device((H, W))
    c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=20, stop_patience=10**9))
    td = nv.to_dev(t, np.uint8)
    L = nv.lib()
    s = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c),
                                    nv.stream(), ctypes.byref(s)))
    nv.check(L.lsopc_session_enqueue(s, 2))
    ms = (ctypes.c_double * 8)()
    nv.check(L.lsopc_session_time_passes(s, 3, ms))
    L.lsopc_session_destroy(s)
    tot = sum(ms)
    print(f"{H}x{W}: {tot:.2f} ms/iter | " + " ".join(f"{n} {v:.2f}" for n, v in zip(NAMES, ms)) +
          f" | per Mpx {tot / (H * W / 1e6):.3f} ms", flush=True)
    del fk, dk
    torch.cuda.empty_cache()
