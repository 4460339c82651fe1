mkdir -p gpurun_out
VARIANTS="default nobar1 row0 pf5 rp c6 c2 rc6" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp3_kbench.log
timeout 1500 python -m pytest tests/test_gpu_c_api.py tests/test_gpu_contract.py tests/test_gpu_engine.py -x -q --durations=5 > gpurun_out/seq_r02d.log 2>&1; echo seq=$?; tail -12 gpurun_out/seq_r02d.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c_api.py --deselect tests/test_gpu_contract.py --deselect tests/test_gpu_engine.py > gpurun_out/gputest_r02d.log 2>&1; echo tests=$?; tail -5 gpurun_out/gputest_r02d.log
