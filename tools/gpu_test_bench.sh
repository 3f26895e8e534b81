# usage: bash tools/gpu_test_bench.sh [pytest -k expr]
set -x
timeout 900 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} 2>&1 | tail -15
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
