# usage: bash tools/gpu_ncu.sh <kernel regex> <tag> [bench args...]
K=$1; TAG=$2; shift 2
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$TAG.log
