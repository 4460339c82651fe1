mkdir -p gpurun_out
VARIANTS="default n54 n18 n36 a27 a9 a27n0" NOPHASES=1 bash tools/vrun.sh 2>&1 | tee gpurun_out/exp5_kbench.log
for v in default cu8 cu16; do
  if [ "$v" = default ]; then L=""; else L="build/libeik_$v.so"; fi
  echo "== $v"; EIK_LIB=$L timeout 120 python tools/phases.py C3 6 2>&1 | head -1
done 2>&1 | tee gpurun_out/exp5_steps.log
echo "== prof"; EIK_LIB=build/libeik_prof.so timeout 200 python tools/phases.py C3 6 2>&1 | tee gpurun_out/exp5_prof.log
echo "== prof mono"; EIK_STEP_MONO=1 EIK_LIB=build/libeik_prof.so timeout 200 python tools/phases.py C3 6 2>&1 | tee -a gpurun_out/exp5_prof.log
