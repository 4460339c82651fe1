mkdir -p gpurun_out
python tools/diag_cb.py > gpurun_out/diag_cb.log 2>&1; echo diag=$?; cat gpurun_out/diag_cb.log
VARIANTS="default edge2 edge3 edge6 pin10 pin20 pin30" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp1_kbench.log
python -m pytest tests -m gpu -q --durations=25 --deselect tests/test_gpu_engine.py::test_engine_accepts_sparse_and_operator_inputs > gpurun_out/gputest_r02c.log 2>&1; echo tests=$?; tail -40 gpurun_out/gputest_r02c.log
