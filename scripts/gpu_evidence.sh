#!/bin/bash
# Round evidence on one B200: per-iteration DRAM traffic (ncu, all launches of
# one iteration), launch list of a short bench run, ncu --set full of the four
# spectral passes.  Outputs in gpurun_out/ (summarised into profiles/ here).
mkdir -p gpurun_out
for P in ${PRECS:-fp32 fp64}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/iter_$P.csv python scripts/prof_iter.py $P > gpurun_out/iter_$P.log 2>&1; echo iter_$P=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fp32.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --no-tier --no-config0 > gpurun_out/ncu_launch.log 2>&1
echo ncu_launch=$?
if [ -n "$FULL" ]; then
for k in ${KERNELS:-TF1Op TF2Op TA1Op TA2Op}; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"${k}" -s 2 -c 1 \
     -o gpurun_out/prof_${k}_fp32 python scripts/prof_iter.py fp32 > gpurun_out/ncu_${k}.log 2>&1; echo ncu_$k=$?
done
fi
