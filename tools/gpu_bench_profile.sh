set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?; tail -2 gpurun_out/bench1.err; cat gpurun_out/bench1.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_step -s 1 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -5 gpurun_out/ncu_full.log
