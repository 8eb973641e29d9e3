#!/bin/bash
# ncu --set full on the spectral passes (one launch each) + launch list of one bench run
mkdir -p gpurun_out
PREC=${PREC:-fp32}
for k in ${KERNELS:-F1Op F2Op A1Op A2Op}; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"${k}" -s 2 -c 1 \
     -o gpurun_out/prof_${k}_${PREC} python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --precision $PREC \
     > gpurun_out/ncu_${k}.log 2>&1; echo ncu_$k=$?
done
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${PREC}.csv \
   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --precision $PREC > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
fi
ls -la gpurun_out
