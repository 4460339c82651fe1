# ncu --set full of the Krylov microbenchmark kernel and of one step kernel
# (same build) for a side-by-side comparison.  usage: bash tools/gpu_prof_cmp.sh TAG
TAG=${1:-cmp}
mkdir -p gpurun_out
KB="python tools/kbench.py C3 40 2"
ST="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$KB > gpurun_out/plain_kb_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_kbench -s 1 -c 1 -o gpurun_out/kb_$TAG $KB > gpurun_out/ncu_kb_$TAG.log 2>&1; echo ncu_kb=$?
$ST > gpurun_out/plain_st_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_step -s 1 -c 1 -o gpurun_out/st_$TAG $ST > gpurun_out/ncu_st_$TAG.log 2>&1; echo ncu_st=$?
