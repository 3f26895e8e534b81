# residual fork A/B on one box: bash tools/gpu_fork_ab.sh [bench args]
for r in 1 2 3; do for f in late early; do
  echo -n "$f: "; FEB200_BENCH_FORK=$f python bench.py --no-cpu-baseline --no-e2e --steps 50 --sub-configs none "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],4), {k: round(v['kernel_ms']['mean'],4) for k,v in d['modes'].items()}, d['graph'], d['clocks']['sm_mhz'])"
done; done
