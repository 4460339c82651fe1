mkdir -p gpurun_out
for v in t128b4 t128c6 t128c2 t96b5 t128nopf5 t128nopfm; do echo "== $v"; EIK_LIB=build/libeik_$v.so timeout 200 python tools/kbench.py C3 40 5 2>&1 | tail -1;  EIK_LIB=build/libeik_$v.so timeout 300 python tools/kbench.py C4:9 40 3 2>&1 | tail -1; done
EIK_LIB=build/libeik_t128b4.so timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
