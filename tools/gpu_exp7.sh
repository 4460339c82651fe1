mkdir -p gpurun_out
VARIANTS="base0 prep base0 prep" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp7_kbench.log
EIK_LIB=build/libeik_prep.so timeout 600 python -m pytest tests/test_gpu_split_step.py tests/test_gpu_golden.py tests/test_gpu_contract.py -x -q 2>&1 | tail -3
