#!/bin/bash
# GPU-box helper: build, run the C3 bench (no CPU baseline / e2e) and print per-level times.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps ${STEPS:-30} "$@" > gpurun_out/qb.log 2>&1 || { tail -20 gpurun_out/qb.log; exit 1; }
python - <<'PY'
import json
d = json.loads(open("gpurun_out/qb.log").read().strip().splitlines()[-1])
print("ms/encode %.3f  frac %.3f" % (d["ms_per_step"], d["roofline"]["frac"]))
for l in d["levels"]:
    print("B=%2d pool %.3f search %.3f exact %d scanned %.4f frac %.3f" % (l["B"], l["ms_pool"], l["ms_search"], l["exact_evals"], l["pairs_scanned"] * 8.0 / max(l["pairs"], 1), l["roof_frac"] or 0))
PY
