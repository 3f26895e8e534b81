set -x
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo rc=$?
tail -c 3000 gpurun_out/bench_c2.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_matrix -s 1 -c 1 -o gpurun_out/prof_c2_matrix $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 1 -c 1 -o gpurun_out/prof_c2_residual $CMD > gpurun_out/ncu_full_res.log 2>&1; echo ncu3=$?
ls -la gpurun_out
