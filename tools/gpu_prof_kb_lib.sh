# usage: bash tools/gpu_prof_kb_lib.sh TAG LIBPATH
TAG=$1; LIB=$2
mkdir -p gpurun_out
CMD="python tools/kbench.py C3 40 2"
EIK_LIB=$LIB $CMD > gpurun_out/plain_$TAG.log 2>&1 && EIK_LIB=$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_swe_kbench -s 1 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
