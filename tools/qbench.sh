#!/bin/bash
# quick C2x64 bench summary (used during kernel work): step time and per-stage times
timeout 300 python bench.py --no-cpu --no-e2e --no-sides --steps 500 "$@" > gpurun_out/qb.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.log").read().strip().splitlines()[-1])
print("step_us", round(d["ms_per_step"] * 1e3, 1), {k: round(v * 1e3, 1) for k, v in d["stages_ms_per_step"].items()},
      "k_points_frac", round(d["roofline"]["frac"], 3))
PY
