# Full checkpoint on one GPU: tests, smoke, default bench (all forms as sub-results, e2e, cpu
# baseline), reference arm, host-overhead tool, launch list, ncu captures.  usage: bash tools/gpu_checkpoint.sh TAG
T=${1:-ck}
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_$T.json 2>&1; echo ref_rc=$?
python tools/host_overhead.py > gpurun_out/host_overhead_C4_P8_$T.json 2>/dev/null; echo ho=$?
python tools/host_overhead.py --config C5 > gpurun_out/host_overhead_C5_P8_$T.json 2>/dev/null
KEEP="${KEEP:-}" bash tools/gpu_ncu_all.sh $T > gpurun_out/ncu_all_$T.log 2>&1; tail -12 gpurun_out/ncu_all_$T.log
