#!/bin/bash
# quick GPU check: gpu tests + cfg5/cfg4 bench lines (no e2e, short cpu baseline)
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --cpu-seconds 1 --no-e2e "$@" > gpurun_out/q5.json 2> gpurun_out/q5.err || tail -5 gpurun_out/q5.err
timeout 300 python bench.py --config 4 --no-cpu-baseline --no-e2e "$@" > gpurun_out/q4.json 2> gpurun_out/q4.err || tail -5 gpurun_out/q4.err
python - <<'PY'
import json
for f in ["gpurun_out/q5.json", "gpurun_out/q4.json"]:
    try:
        d = json.load(open(f))
        r = d["roofline"]
        print(f, "ms/step %.3f" % d["ms_per_step"], "value %.3e" % d["value"], "kernel_ms %.3f" % r["kernel_ms"],
              "frac %.3f" % r["frac"], "step_frac %.3f" % r["step_frac"], "run_ms %.3f" % d["run_ms_device"], d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
