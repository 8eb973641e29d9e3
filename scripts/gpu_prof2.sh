./scripts/microbench_colaccess > gpurun_out/microbench_col.txt 2>&1; cat gpurun_out/microbench_col.txt
for k in FFwdCol FAdjCol FFwdRow; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$k -s 30 -c 1 -o gpurun_out/prof2_$k python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu2_$k.log 2>&1; echo ncu_$k=$?
done
