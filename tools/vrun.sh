# usage: VARIANTS="a b" bash tools/vrun.sh   -- Krylov microbenchmark + step time per build/libeik_<v>.so
for v in ${VARIANTS}; do
  if [ "$v" = default ]; then L=""; else L="build/libeik_$v.so"; fi
  echo "== $v"; EIK_LIB=$L timeout 120 python tools/kbench.py C3 40 5 2>&1 | tail -2
  [ -n "$NOPHASES" ] || EIK_LIB=$L timeout 120 python tools/phases.py C3 6 2>&1 | head -1
done
