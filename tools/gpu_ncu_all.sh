# ncu evidence for every BASELINE kernel (one --set full capture each) plus the launch list of
# the default bench command.  usage: bash tools/gpu_ncu_all.sh <tag>
T=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sub-configs none --clock-window 0"
cap() {  # cap <kernel regex> <name> <bench args...>
  local K=$1 N=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o /tmp/prof_${T}_$N $B "$@" > gpurun_out/ncu_${T}_$N.log 2>&1; echo "$N ncu=$?"
}
$B > gpurun_out/plain_$T.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${T}_C2.csv $B > gpurun_out/ncu_${T}_launch.log 2>&1; echo launch=$?
cap "k_matrix_sfp" C2_matrix --config C2
cap "k_residual_t3" C2_residual --config C2
cap "k_matrix_vp" C3_matrix --config C3
cap "k_residual_t3e" C3_residual --config C3
cap "k_residual_sf" C4_residual_f64 --config C4
cap "k_residual_sf" C4_residual_f32 --config C4 --dtype f32
cap "k_residual_t3c" C5_residual --config C5
cap "k_matrix_vp" C5t_matrix --config C5t
cap "k_matrix_vp" C3d_matrix --config C3d
cap "k_assemble_matrix" C2csr_assembly --config C2csr
cap "k_assemble_matrix" C3csr_assembly --config C3csr
# summaries (and the raw csv pages) come back; the reports stay in /tmp except the ones named
# in KEEP (gpurun_out/ is capped at 64 MiB)
for f in /tmp/prof_${T}_*.ncu-rep; do
  b=$(basename ${f%.ncu-rep})
  python tools/ncu_summary.py $f > gpurun_out/$b.txt 2>&1
  ncu -i $f --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
done
for k in $KEEP; do cp /tmp/prof_${T}_$k.ncu-rep gpurun_out/ 2>/dev/null; done
du -sh gpurun_out
