#!/bin/bash
# GPU box: C3 bench of the default build and of each abvar/*.so under the large-s modes
for mode in ${MODES:-grid sampled10 closed5}; do
for so in default $(ls abvar/*.so 2>/dev/null); do
  if [ "$so" = default ]; then unset FIC_SO; else export FIC_SO=$PWD/$so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --s-mode $mode --steps ${STEPS:-20} > gpurun_out/abm.log 2>&1 || { echo "$mode $so failed"; tail -3 gpurun_out/abm.log; continue; }
  python - "$mode" "$so" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/abm.log").read().strip().splitlines()[-1])
print("%-10s %-16s ms/encode %.4f " % (sys.argv[1], sys.argv[2], d["ms_per_step"]) + " ".join("B%d %.4f" % (l["B"], l["ms_search"]) for l in d["levels"]) + "  B2 scanned %.3f" % (1 - d["levels"][-1]["pruned_frac"]))
PY
done; done
