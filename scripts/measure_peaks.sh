#!/bin/bash
# GPU box: measure the pair-kernel roofline denominators (scripts/micro/peaks.cu) and write them
# to gpurun_out/peaks.json (copied to profiles/peaks_r02.json, which bench.py reads).
set -e
cd "$(dirname "$0")/micro"
mkdir -p bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/peaks peaks.cu
cd ../..
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > gpurun_out/peaks_smi_before.txt
scripts/micro/bin/peaks > gpurun_out/peaks_raw.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader > gpurun_out/peaks_smi_after.txt
python - <<'PY'
import json, subprocess
d = json.load(open("gpurun_out/peaks_raw.json"))
d["how"] = ("scripts/micro/peaks.cu: every SM at full occupancy (int/fp64: 4 x 512 threads per SM, 8 "
            "independent chains per thread; int8: one CTA per SM, one thread issuing tcgen05.mma "
            "kind::i8 M=128 N=256 K=32 into two TMEM accumulators), CUDA events, best of 5")
d["smi_before"] = open("gpurun_out/peaks_smi_before.txt").read().strip()
d["smi_after"] = open("gpurun_out/peaks_smi_after.txt").read().strip()
json.dump(d, open("gpurun_out/peaks.json", "w"), indent=1)
print(json.dumps(d, indent=1))
PY
