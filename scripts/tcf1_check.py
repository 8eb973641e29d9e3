"""Tensor-core F1 (f1_tc.cu) (opt-in, LSOPC_B200_TCF1=1) against the FFT F1 (default) and the
float64 tier on the same inputs (dev check): intensity at the three corners
and the ILT gradient on the 2048^2 clip, 24 + 24 kernels."""
import json
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv, inputs
    nv.set_precision(sys.argv[2])
    clip = inputs.iccad_like_clip(seed=0).astype(np.float64)
    f, d = b2.gen_synthetic_kernels(35, 24, seed=4)
    out = {}
    for name, ks, cond in (("nom", f, b2.NOMINAL), ("out", f, b2.OUTER), ("in", d, b2.INNER)):
        out[name] = b2.aerial_intensity(clip, ks, cond)
    z = b2.print_corners(clip, f, d, b2.OptConfig(), binarize=False).nominal
    out["g"] = b2.ilt_gradient(clip, z, clip.astype(np.uint8), f, b2.OptConfig())
    np.savez(sys.argv[3], **out)
    sys.exit(0)
import numpy as np
runs = {"tc": ("fp32", {"LSOPC_B200_TCF1": "1"}), "fft": ("fp32", {}), "f64": ("fp64", {})}
for tag, (prec, env) in runs.items():
    p = subprocess.run([sys.executable, __file__, "run", prec, f"/tmp/tcf1_{tag}.npz"], env={**os.environ, **env},
                       capture_output=True, text=True)
    if p.returncode:
        print(tag, "FAILED", p.stderr[-3000:])
        sys.exit(1)
r = {t: np.load(f"/tmp/tcf1_{t}.npz") for t in runs}
res = {}
for k in ("nom", "out", "in", "g"):
    ref = r["f64"][k]
    res[k] = {t: float(np.abs(r[t][k] - ref).max() / np.abs(ref).max()) for t in ("tc", "fft")}
print(json.dumps(res, indent=1))
