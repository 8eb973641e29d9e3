import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import dsn, inputs, _native as nv
ts = [inputs.iccad_like_clip(seed=500 + i) for i in range(16)]
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x = dsn.tsdf_batch(ts)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"tsdf_batch 16: {1e3*(t1-t0):.1f} ms")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    b2.tsdf_from_mask(ts[0])
    torch.cuda.synchronize(); print(f"tsdf_from_mask: {1e3*(time.perf_counter()-t0):.1f} ms")
