# ad-hoc A/B: parity of every variant on the given pytest -k expression, then timing per config
# usage: bash tools/gpu_ab_ad.sh "<pytest -k expr>" CONFIG...
K="$1"; shift
for lib in paper_2107_04121_b200/ab/lib_*.so; do
  v=$(basename $lib .so); echo -n "${v#lib_} parity: "
  FEB200_LIB_PATH=$PWD/$lib timeout 900 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -1
done
for c in "$@"; do bash tools/gpu_ab.sh --config $c; done
