# bench every workload once (device-timed, no e2e / cpu baseline) -> gpurun_out/configs.jsonl
: > gpurun_out/configs.jsonl
for c in C1 C2 C3 C4 C5 C5t C2csr C3csr C3d; do
  python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e --sub-configs none >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err || echo "fail $c" >> gpurun_out/configs.err
done
python bench.py --config C4 --dtype f32 --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err || echo "fail C4f32" >> gpurun_out/configs.err
python bench.py --config C2 --dtype f32 --steps 20 --no-cpu-baseline --no-e2e --sub-configs none >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err || echo "fail C2f32" >> gpurun_out/configs.err
python bench.py --config C2 --fused --steps 20 --no-cpu-baseline --no-e2e >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err || echo "fail C2fused" >> gpurun_out/configs.err
FEB200_RESIDUAL_IMPL=dense FEB200_MATRIX_IMPL=dense python bench.py --config C2 --steps 20 --no-cpu-baseline --no-e2e --sub-configs none >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
tail -3 gpurun_out/configs.err
