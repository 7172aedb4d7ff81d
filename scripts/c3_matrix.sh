#!/bin/bash
# GPU box: the C3 measurement matrix (BASELINE.json configs[2]): t in {4, 8, 12} x {predefined, grid},
# full bench lines (oracle parity + cpu_baseline included) -> gpurun_out/c3_<mode>_t<t>.json
for mode in predefined grid; do
  for t in 4 8 12; do
    timeout 600 python bench.py --s-mode $mode --t $t --steps ${STEPS:-30} > gpurun_out/c3_${mode}_t${t}.log 2>&1
    tail -1 gpurun_out/c3_${mode}_t${t}.log > gpurun_out/c3_${mode}_t${t}.json
    python - "$mode" "$t" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/c3_{sys.argv[1]}_t{sys.argv[2]}.json"))
print("%-10s t=%-2s ms/encode %.3f parity %s  " % (sys.argv[1], sys.argv[2], d["ms_per_step"], d.get("parity", {}).get("bit_exact_all_fields")) +
      " ".join("B%d %.3f" % (l["B"], l["ms_search"]) for l in d["levels"]))
PY
  done
done
