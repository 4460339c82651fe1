# bench + reference arm + launch list + one full ncu capture each of the Krylov sweep kernel,
# the continuation kernel and the dense phi kernel; TAG as $1
# (ncu passes run with EIK_STEP_HOST=1: kernels inside conditional graph nodes cannot be profiled;
#  EIK_SWEEP_LOG=1 prints each sweep's Krylov iteration count to match the captured launch)
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
[ -n "$NOREF" ] || { python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref=$?; }
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --sweep-steps 2"
export EIK_STEP_HOST=1 EIK_SWEEP_LOG=1
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo ncu1=$?
# capture a full-length sweep: the first launch with >= 30 Krylov iterations in the plain run
KSKIP=${KSKIP:-$(python -c "
import re,sys
for l in open('gpurun_out/plain_$TAG.log'):
    m = re.match(r'\[eik\] sweep (\d+) iters (\d+)', l)
    if m and int(m.group(2)) >= 30:
        print(m.group(1)); break
")}
echo "KSKIP=$KSKIP" > gpurun_out/kskip_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_sweep -s $KSKIP -c 1 -o gpurun_out/step_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu2=$?
[ -n "$NOCONT" ] || { timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_cont -s 3 -c 1 -o gpurun_out/cont_$TAG $CMD > gpurun_out/ncu_cont_$TAG.log 2>&1; echo ncu3=$?; }
[ -n "$NOCONT" ] || { timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_dense -s 3 -c 1 -o gpurun_out/dense_$TAG $CMD > gpurun_out/ncu_dense_$TAG.log 2>&1; echo ncu4=$?; }
