# A/B timing of every variant build in paper_2107_04121_b200/ab/ (tools/build_ab.py) on the
# same box, interleaved twice:  bash tools/gpu_ab.sh [bench args]
for r in 1 2; do for lib in paper_2107_04121_b200/ab/lib_*.so; do
  v=$(basename $lib .so); echo -n "${v#lib_}: "
  FEB200_LIB_PATH=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 \
    --sub-configs none --clock-window 0 "$@" 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(d['config']['workload'], ' '.join(f\"{k} {v['kernel_ms']['mean']:.4f} ms\" for k, v in d['modes'].items()))"
done; done
