#!/bin/bash
# round-1 GPU pass: parity tests, bench (both tiers), launch list
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo bench32_rc=$?
timeout 600 python bench.py --no-cpu-baseline --no-solve --precision fp64 > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err; echo bench64_rc=$?
cat gpurun_out/bench_fp32.json gpurun_out/bench_fp64.json; tail -5 gpurun_out/bench_fp32.err gpurun_out/bench_fp64.err
