mkdir -p gpurun_out
for v in default n54 nopf5 c6 c6n54 t128c6 default; do
  if [ "$v" = default ]; then L=""; else L="build/libeik_$v.so"; fi
  EIK_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/b15_${v}.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/b15_${v}.json"))
print("$v", "value %.2f ms %.3f us/iter %.2f frac %.4f step_frac %.4f day %.2f e2e %.2f" % (d["value"], d["ms_per_step"], d["roofline"]["us_per_iter"], d["roofline"]["frac"], d["roofline"]["step_frac"], d["full_run"]["steps_per_s"], d["e2e"]["value"]))
PY
done
