# bench lines beyond the headline: EPI3 on C3, EXPRB4 / EXPRB5 on C4 at L9 and L10 (TAG as $1)
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --scheme epi3 --no-cpu-baseline > gpurun_out/bench_c3_epi3_$TAG.json 2> gpurun_out/bench_c3_epi3_$TAG.err; echo epi3=$?
for L in 9 10; do
  for S in exprb42 exprb53; do
    timeout 1200 python bench.py --config C4 --level $L --scheme $S --steps 10 --warmup 3 --no-cpu-baseline \
      > gpurun_out/bench_c4_l${L}_${S}_$TAG.json 2> gpurun_out/bench_c4_l${L}_${S}_$TAG.err; echo l$L$S=$?
  done
done
