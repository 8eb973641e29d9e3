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
# device-only: lsopc_tsdf on resident buffers, CUDA events
for i in (0, 1):
    td = nv.to_dev(np.ascontiguousarray((ts[i] != 0).astype(np.uint8)), np.uint8)
    phi = nv.empty(ts[i].shape, np.float64)
    H, W = ts[i].shape
    call = lambda: nv.check(nv.lib().lsopc_tsdf(H, W, nv.ptr(td), 900.0, -100.0, nv.ptr(phi), nv.stream()))
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()  # nv.stream() is the current stream
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        call()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"lsopc_tsdf device {H}x{W} clip {i}: {e0.elapsed_time(e1) / 20 * 1e3:.0f} us")
