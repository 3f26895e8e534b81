# end-of-session checkpoint on one GPU: tests, smoke, default bench, reference arm, launch list
# of the default bench command.  usage: bash tools/gpu_final.sh TAG
T=${1:-fin}
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_$T.json 2>&1; echo ref_rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sub-configs none --clock-window 0"
$B > gpurun_out/plain_$T.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${T}_C2.csv $B > gpurun_out/ncu_${T}_launch.log 2>&1; echo launch=$?
