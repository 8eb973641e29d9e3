"""Tall-grid column passes: split plan / cluster paths vs the single-column path (dev check).
Prints max relative difference of the loss history and the final-mask XOR."""
import json, os, subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import inputs
    H, W = int(sys.argv[2]), int(sys.argv[3])
    clip = np.ascontiguousarray(inputs.mosaic_tile(range(16), grid=(4, 4))[:H, 3000:3000 + W])
    (fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
    F = b2.KernelSet([b2.OpticalKernel(c, float(x)) for c, x in zip(fc, fw)], "focus")
    D = b2.KernelSet([b2.OpticalKernel(c, float(x)) for c, x in zip(dc, dw)], "defocus")
    r = b2.optimize(clip, F, D, b2.OptConfig(max_iters=6, stop_patience=10**9, precision="fp32"))
    np.save(sys.argv[4], r.final_mask)
    print(json.dumps([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v] for h in r.loss_history]))
    sys.exit(0)
import numpy as np
H, W = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (8192, 256)
out = {}
extra = sys.argv[3] if len(sys.argv) > 3 else ""          # e.g. LSOPC_B200_NO_VSPLIT=1,LSOPC_B200_NO_SPLIT=1
env_extra = dict(kv.split("=") for kv in extra.split(",") if kv)
# reference leg: the single-column cp.async column passes of the unsplit plan
single = {"LSOPC_B200_NO_CLUSTER": "1", "LSOPC_B200_NO_VSPLIT": "1"}
for tag, env in (("cluster", env_extra), ("single", single)):
    p = subprocess.run([sys.executable, __file__, "run", str(H), str(W), f"/tmp/cc_{tag}.npy"], capture_output=True,
                       text=True, env={**os.environ, **env})
    if p.returncode:
        print(tag, "FAILED", p.stderr[-3000:]); sys.exit(1)
    out[tag] = np.array(json.loads(p.stdout.strip().splitlines()[-1]))
rel = np.abs(out["cluster"] - out["single"]).max(axis=0) / np.abs(out["single"]).max(axis=0)
xor = int((np.load("/tmp/cc_cluster.npy") != np.load("/tmp/cc_single.npy")).sum())
print(f"{H}x{W}: history max rel diff {rel.max():.3e}, final mask xor {xor}")
