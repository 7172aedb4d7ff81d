#!/bin/bash
# GPU box: C3 bench (no parity) of the default build and each abvar/*.so, with per-level search
# times and exact-path counts (timing diagnostics may change the filter's pass counts)
for so in default $(ls abvar/*.so 2>/dev/null); do
  if [ "$so" = default ]; then unset FIC_SO; else export FIC_SO=$PWD/$so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps ${STEPS:-30} "$@" > gpurun_out/ab.log 2>&1 || { echo "$so failed"; tail -3 gpurun_out/ab.log; continue; }
  python - "$so" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
print("%-22s ms/encode %.4f " % (sys.argv[1], d["ms_per_step"]) + " ".join("B%d %.4f x%d" % (l["B"], l["ms_search"], l["exact_evals"]) for l in d["levels"]))
PY
done
