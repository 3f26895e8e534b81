# Full checkpoint on one GPU: tests, default bench (with e2e + cpu baseline), all configs,
# reference arm, ncu launch list and one --set full capture of the dominant kernel.
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench_rc=$?
cat gpurun_out/bench_default.json
bash tools/gpu_all_configs.sh
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; echo ref_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_ck.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ck.csv $CMD > gpurun_out/ncu_ck_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_matrix_sfp -s 1 -c 1 -o gpurun_out/prof_ck_matrix $CMD > gpurun_out/ncu_ck_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_residual_t3 -s 1 -c 1 -o gpurun_out/prof_ck_residual $CMD > gpurun_out/ncu_ck_full_r.log 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:k_matrix_vp -s 1 -c 1 -o gpurun_out/prof_ck_c3_matrix python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ck_c3.log 2>&1; echo ncu4=$?
ncu --set full --clock-control none --import-source on -k regex:k_residual_t3c -s 1 -c 1 -o gpurun_out/prof_ck_c5_residual python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ck_c5.log 2>&1; echo ncu5=$?
