"""Instant-OPC DSO stage, per-clip call times (dev probe)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, dsn, inputs  # noqa: E402
from paper_2303_12529_b200.optimizer import _optimize_device  # noqa: E402

nv.set_precision("fp32")
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
cfg = b2.OptConfig(precision="fp32")
net = dsn.build_net()
dsn.instant_opc([inputs.iccad_like_clip(seed=900)], focus, defocus, cfg, net=net)
targets = [inputs.iccad_like_clip(seed=500 + i) for i in range(16)]
for rep in range(2):
    r = dsn.instant_opc(targets, focus, defocus, cfg, net=net)
    print(f"rep {rep}: tsdf {r.t_tsdf:.4f} net {r.t_net:.4f} init {r.t_init:.4f} dso {r.t_dso:.4f} "
          f"iters {sum(x.iters_run for x in r.results)}", flush=True)
x = dsn.tsdf_batch(targets, cfg.d_upper, cfg.d_lower)
with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
    phi_raw, m_raw = net((x / 100.0).float().unsqueeze(1))
phi0, m = dsn.dsn_init(x.float() + 100.0 * phi_raw.float().squeeze(1), m_raw.float().squeeze(1), cfg)
ts = []
for i, t in enumerate(targets):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = _optimize_device(t, focus, defocus, cfg, phi0=phi0[i], modulation=m[i])
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0, p))
print(" ".join(f"{1e3 * a:.1f}" for a, _ in ts))
