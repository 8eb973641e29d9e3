set -x
nproc; lscpu | grep "Model name"; free -g | head -2
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1_rc=$?
for k in FFwdCol FFwdRow FAdjRow FAdjCol; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$k -s 30 -c 1 -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_$k.log 2>&1; echo ncu_$k=$?
done
ls -la gpurun_out
