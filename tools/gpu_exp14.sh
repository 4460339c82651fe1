mkdir -p gpurun_out
for r in 1 2; do for v in 0 1; do
  EIK_TILECOEF=$v python bench.py --no-cpu-baseline > gpurun_out/b14_${v}_$r.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/b14_${v}_$r.json"))
print("tilecoef=$v", $r, "value %.2f ms %.3f us/iter %.2f frac %.4f step_frac %.4f day %.2f e2e %.2f" % (d["value"], d["ms_per_step"], d["roofline"]["us_per_iter"], d["roofline"]["frac"], d["roofline"]["step_frac"], d["full_run"]["steps_per_s"], d["e2e"]["value"]))
PY
done; done
for v in 0 1; do echo "== tilecoef $v"; EIK_TILECOEF=$v python tools/kbench.py C3 40 5 | tail -1; EIK_TILECOEF=$v python tools/kbench.py C4:9 40 3 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_split_step.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_planar_steps.py tests/test_gpu_swe_api.py -x -q 2>&1 | tail -3
