#!/bin/bash
# GPU box: C3 bench of the default build under each environment setting given as an argument
# (e.g. "FIC_SIDE_PRIO=hi"), twice each, interleaved
for rep in 1 2; do
for envs in "" "$@"; do
  ( [ -n "$envs" ] && export $envs; timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps ${STEPS:-30} > gpurun_out/abe.log 2>&1 ) || { echo "$envs failed"; continue; }
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abe.log").read().strip().splitlines()[-1])
print("%-26s ms/encode %.4f " % (sys.argv[1] or "default", d["ms_per_step"]) + " ".join("B%d %.4f" % (l["B"], l["ms_search"]) for l in d["levels"]))
PY
done; done
