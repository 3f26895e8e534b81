# A/B timing of alternative builds on the same box: bash tools/gpu_ab.sh [bench args]
for r in 1 2; do for v in A B; do
  echo -n "$v: "; FEB200_LIB_PATH=$PWD/paper_2107_04121_b200/ab/lib_$v.so python bench.py --no-cpu-baseline --no-e2e --steps 30 "$@" 2>/dev/null | grep -o '"modes": {[^}]*}[^}]*}'
done; done
