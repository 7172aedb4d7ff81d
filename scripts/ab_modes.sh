#!/bin/bash
# GPU box: C3 bench of the default build under the large-s modes, with and without the given
# environment setting (e.g. FIC_B2_WINK=0), interleaved
for rep in 1 2; do
for mode in grid sampled10 closed5; do
for envs in "" "$@"; do
  ( [ -n "$envs" ] && export $envs; timeout 300 python bench.py --no-cpu-baseline --no-e2e --s-mode $mode --steps ${STEPS:-20} > gpurun_out/abm.log 2>&1 ) || { echo "$mode $envs failed"; tail -3 gpurun_out/abm.log; continue; }
  python - "$mode" "$envs" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abm.log").read().strip().splitlines()[-1])
print("%-10s %-16s ms/encode %.4f " % (sys.argv[1], sys.argv[2] or "default", d["ms_per_step"]) + " ".join("B%d %.4f" % (l["B"], l["ms_search"]) for l in d["levels"]) + "  B2 scanned %.3f" % (1 - d["levels"][-1]["pruned_frac"]))
PY
done; done; done
