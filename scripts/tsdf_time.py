import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch, ctypes
from paper_2303_12529_b200 import _native as nv, inputs
clip = inputs.iccad_like_clip(seed=0)
td = nv.to_dev(clip, np.uint8); out = nv.empty(clip.shape, np.float64)
L = nv.lib()
for rep in range(3):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    nv.check(L.lsopc_tsdf(2048, 2048, nv.ptr(td), 900.0, -100.0, nv.ptr(out), nv.stream()))
    e1.record(); torch.cuda.synchronize(); print(f"tsdf 2048^2: {e0.elapsed_time(e1):.3f} ms (incl. uniform check + sync)")
