mkdir -p gpurun_out
for r in 1 2; do for v in default t256 t256c6 t128c3; do
  if [ "$v" = default ]; then L=""; else L="build/libeik_$v.so"; fi
  EIK_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/b13_${v}_$r.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/b13_${v}_$r.json"))
print("$v", $r, "value %.2f ms %.3f us/iter %.2f frac %.4f step_frac %.4f day %.2f e2e %.2f" % (d["value"], d["ms_per_step"], d["roofline"]["us_per_iter"], d["roofline"]["frac"], d["roofline"]["step_frac"], d["full_run"]["steps_per_s"], d["e2e"]["value"]))
PY
done; done
