for v in ${VARIANTS:-tma256b1 tma128b2 tma128b3 t256b2}; do
  echo "== $v"; EIK_LIB=build/libeik_$v.so timeout 120 python tools/kbench.py C3 40 5 2>&1 | tail -2
done
