#!/bin/bash
# Round evidence: default bench line, ncu launch list, ncu --set full of the dominant pass.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -3 gpurun_out/bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fp32.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --clips 0 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
for k in ${KERNELS:-TA2Op TF2Op}; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"${k}" -s 2 -c 1 \
   -o gpurun_out/prof_${k}_fp32 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --clips 0 \
   > gpurun_out/ncu_${k}.log 2>&1; echo ncu_$k=$?
done
