mkdir -p gpurun_out
for x in 0 1 2; do echo "== t128b4 extra $x"; EIK_TILES_EXTRA=$x EIK_LIB=build/libeik_t128b4.so timeout 200 python tools/kbench.py C3 40 5 2>&1 | tail -2; done
for x in 1 2; do echo "== default extra $x"; EIK_TILES_EXTRA=$x timeout 200 python tools/kbench.py C3 40 5 2>&1 | tail -2; done
echo "== t128b4 L9"; EIK_LIB=build/libeik_t128b4.so timeout 300 python tools/kbench.py C4:9 40 3 2>&1 | tail -1
echo "== t128b4 step"; EIK_LIB=build/libeik_t128b4.so timeout 200 python tools/phases.py C3 6 2>&1 | head -1
echo "== default step"; timeout 200 python tools/phases.py C3 6 2>&1 | head -1
