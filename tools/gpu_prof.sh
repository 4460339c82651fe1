# usage: bash tools/gpu_prof.sh <tag>
TAG=${1:-prof}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_step -s 1 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$TAG.log
