# compute-sanitizer passes over the small-size GPU parity tests (every kernel family, ragged
# batches, misaligned views, capped grids).  usage: bash tools/gpu_sanitize.sh TAG
# memcheck: out-of-bounds / misaligned accesses of global, shared and local memory, API errors;
# synccheck: invalid barrier / mbarrier use; racecheck: shared-memory hazards (reported only:
# it does not model bulk-async copies completing on an mbarrier).
T=${1:-san}
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
K1="single_cell or pipelined_many_batches or n3_n4_many or residual_misaligned or unaligned_outputs or matrix_q4 or matrix_fp32 or residual_fp32 or matrix_residual_fused or stress or stokes_coupling or eval_mode or csr_assembly or full_d_nonsymmetric or element_ranges or assemble_vector or geometry_materialized or weighted_dot or elasticity_material or mixed_order or group_cells"
K2="single_cell or pipelined_many_batches or n3_n4_many or residual_fp32"
run() { # tool, -k expr, time limit
  local tool=$1 k=$2 lim=$3
  timeout $lim compute-sanitizer --tool $tool --error-exitcode 86 --print-limit 20 \
    --log-file gpurun_out/sanitize_${T}_$tool.log \
    python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$k" \
    > gpurun_out/sanitize_${T}_$tool.pytest 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_${T}_$tool.pytest
  grep -c "=========" gpurun_out/sanitize_${T}_$tool.log; tail -3 gpurun_out/sanitize_${T}_$tool.log
}
run memcheck "$K1" 1500
run synccheck "$K2" 900
run racecheck "$K2" 900
