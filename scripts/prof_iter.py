"""Run W + K DSO iterations of the bench workload (2048^2 iccad_like_clip,
24 + 24 kernels) in one session, for ncu:
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/iter_fp32.csv python scripts/prof_iter.py fp32
then `python scripts/prof_iter.py --summarise gpurun_out/iter_fp32.csv fp32` writes
profiles/traffic_<prec>.json (DRAM bytes per launch of one iteration, by pass)."""
import csv
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PASSES = [("mask_fft", ("TMaskRowsOp", "TColsOp", "MaskRowsOp", "ColsOp")), ("F1", ("TF1Op", "F1COp", "F1Op")),
          ("F2", ("TF2Op", "F2Op")), ("resist", ("k_resist", "k_copy_best")), ("A1", ("TA1Op", "A1Op")),
          ("A2", ("TA2Op", "A2Op")), ("A3", ("A3Op",)), ("levelset", ("k_ls_velocity", "k_ls_update"))]


def run(prec, W=3, K=2, shape=None):
    import numpy as np
    import torch
    import paper_2303_12529_b200 as b2
    from paper_2303_12529_b200 import _native as nv, inputs
    nv.set_precision(prec)
    if shape is None:
        clip = inputs.iccad_like_clip(seed=0)
    else:  # another geometry (e.g. a split plan): a crop of the configs[4] mosaic
        H, Wd = shape
        clip = np.ascontiguousarray(inputs.mosaic_tile(range(16), grid=(4, 4))[:H, 2048:2048 + Wd])
    focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
    fk, dk = focus.device(clip.shape, prec), defocus.device(clip.shape, prec)
    c = b2.optimizer._native_cfg(b2.OptConfig(max_iters=W + K + 2, stop_patience=10**9, precision=prec))
    td = nv.to_dev(clip, np.uint8)
    L = nv.lib()
    s = ctypes.c_void_p()
    nv.check(L.lsopc_session_create(fk.plan.handle, fk.handle, dk.handle, nv.ptr(td), None, None, ctypes.byref(c),
                                    nv.stream(), ctypes.byref(s)))
    nv.check(L.lsopc_session_enqueue(s, W + K))
    torch.cuda.synchronize()
    print("launches per iteration", L.lsopc_session_launches_per_iter(s))
    L.lsopc_session_destroy(s)


def summarise(path, prec, per_iter=11, tag=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hd = rows[h]
    ki, mi, vi, ii = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value"), hd.index("ID")
    launches = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(launches)
    last = [launches[i] for i in ids[-per_iter:]]
    out = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"(one launch each, cold-cache replay) of the last DSO iteration of scripts/prof_iter.py {prec}",
           "launches": []}
    total = 0.0
    per_pass = {str(i): 0.0 for i in range(len(PASSES))}
    for d in last:
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        total += b
        idx = next((i for i, (_, tags) in enumerate(PASSES) if any(t in d["name"] for t in tags)), None)
        if idx is not None:
            per_pass[str(idx)] += b
        out["launches"].append({"kernel": d["name"][:90], "pass": PASSES[idx][0] if idx is not None else None,
                                "us": round(d.get("gpu__time_duration.sum", 0.0) / 1e3, 2), "dram_bytes": b})
    out["iteration"] = total
    out.update(per_pass)
    out["pass_names"] = {str(i): n for i, (n, _) in enumerate(PASSES)}
    dst = ROOT / "profiles" / f"traffic_{tag or prec}.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--summarise":  # --summarise <csv> <prec> [tag]
        summarise(sys.argv[2], sys.argv[3], tag=sys.argv[4] if len(sys.argv) > 4 else None)
    else:  # <prec> [H W]
        run(sys.argv[1], shape=(int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else None)
