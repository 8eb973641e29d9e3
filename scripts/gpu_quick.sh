# quick perf check: pytest subset + bench both tiers (no CPU baseline / solve)
timeout 600 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-solve > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo bench32_rc=$?
timeout 300 python bench.py --no-cpu-baseline --no-solve --precision fp64 > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo bench64_rc=$?
python - <<'PY'
import json
for p in ("fp32","fp64"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{p}.json").read().strip().splitlines()[-1])
        print(p, d["value"], "iters/s", d["ms_per_step"], "ms;", {k:(v["us"],v["frac"]) for k,v in d["roofline"]["per_pass"].items()}, "e2e", d["e2e"]["value"])
    except Exception as e: print(p, "ERR", e); print(open(f"gpurun_out/bench_{p}.err").read()[-2000:])
PY
