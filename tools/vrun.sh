for v in s256b2 s128b4 s128b3 s512b1 s256b1 s384b1 s256b2c2 s256b2c6; do
  echo "== $v"; EIK_LIB=build/libeik_$v.so timeout 120 python tools/kbench.py C3 40 5 2>&1 | tail -1
done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | cut -c1-200
for v in s256b2 s128b4 s256b1; do echo "== $v"; EIK_LIB=build/libeik_$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | cut -c1-200; done
