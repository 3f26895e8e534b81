# Parity of every A/B variant (matrix tests of the vector forms) then the A/B timing.
# usage: bash tools/gpu_ab_parity.sh "<pytest -k expr>" [bench args]
K=$1; shift
for lib in paper_2107_04121_b200/ab/lib_*.so; do
  v=$(basename $lib .so); echo -n "${v#lib_} parity: "
  FEB200_LIB_PATH=$PWD/$lib timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -1
done
bash tools/gpu_ab.sh "$@"
