mkdir -p gpurun_out
VARIANTS="base0 prep base0 prep" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp6_kbench.log
EIK_LIB=build/libeik_prep.so python -m pytest tests/test_gpu_split_step.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
