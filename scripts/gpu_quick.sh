#!/bin/bash
# quick perf check: pytest gpu subset + bench both tiers (no CPU baseline / solve)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -25 gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-solve > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo bench32_rc=$?
timeout 300 python bench.py --no-cpu-baseline --no-solve --precision fp64 > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo bench64_rc=$?
python - <<'PY'
import json
for p in ("fp32","fp64"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{p}.json").read().strip().splitlines()[-1])
        print(p, d["value"], "iters/s", d["ms_per_step"], "ms; e2e", d["e2e"]["value"])
        for k,v in d["roofline"]["per_pass"].items(): print("   %-60s %9.1f us %7.1f GB/s %.3f" % (k, v["us"], v["GBps"], v["frac"]))
        print("   iteration", d["roofline"]["iteration"])
    except Exception as e: print(p, "ERR", e); print(open(f"gpurun_out/bench_{p}.err").read()[-3000:])
PY
