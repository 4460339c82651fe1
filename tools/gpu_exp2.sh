mkdir -p gpurun_out
VARIANTS="default half2 bar1 bh pre3 bp bph" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp2_kbench.log
for k in 1 2 3; do
  python -m pytest tests/test_gpu_c_api.py tests/test_gpu_contract.py tests/test_gpu_engine.py -x -q > gpurun_out/flaky_$k.log 2>&1; echo flaky$k=$?; tail -3 gpurun_out/flaky_$k.log
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_engine.py -x -q -k "dense_oracle or counters or accepts or callable_operator_matches or full_dimension" > gpurun_out/initcheck.log 2>&1; echo initcheck=$?; grep -c "Uninitialized" gpurun_out/initcheck.log; tail -5 gpurun_out/initcheck.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_engine.py -x -q -k "dense_oracle or counters or accepts or callable_operator_matches or full_dimension" > gpurun_out/memcheck.log 2>&1; echo memcheck=$?; tail -5 gpurun_out/memcheck.log
