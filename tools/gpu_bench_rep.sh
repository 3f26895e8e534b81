# usage: bash tools/gpu_bench_rep.sh N [bench args]
N=$1; shift
for i in $(seq $N); do python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | grep -o '"modes": {[^}]*}[^}]*}'; done
