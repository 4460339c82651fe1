# bench + launch list + one full ncu capture of the step kernel; TAG as $1
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref=$?
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_step -s 1 -c 1 -o gpurun_out/step_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2=$?
