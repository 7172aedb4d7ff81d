#!/bin/bash
# GPU box, round 2 final refresh: every committed result line (scripts/refresh_results_r02.sh),
# then the ncu captures of scripts/refresh_profiles_r02.sh reusing those bench lines.
set -x
bash scripts/refresh_results_r02.sh
cp gpurun_out/r02/bench_c3.json gpurun_out/bench_r02.log
cp gpurun_out/r02/bench_c4.json gpurun_out/bench_c4_r02.log
cp gpurun_out/r02/bench_c5.json gpurun_out/bench_c5_r02.log
cp gpurun_out/r02/launches.csv gpurun_out/launches_r02.csv
mkdir -p /tmp/reps
timeout 1200 ncu --set full --clock-control none --launch-skip 60 --launch-count 70 \
    -f -o /tmp/reps/prof_c3_r02 python scripts/one_encode.py C3 1 > gpurun_out/ncu_c3_r02.log 2>&1
ncu -i /tmp/reps/prof_c3_r02.ncu-rep --page raw --csv > gpurun_out/prof_c3_r02_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"entropy|pool|select_chain|t2f|ctab" --launch-skip 15 --launch-count 15 \
    -f -o /tmp/reps/prof_c5pool_r02 python scripts/one_encode.py C5 1 > gpurun_out/ncu_c5pool_r02.log 2>&1
ncu -i /tmp/reps/prof_c5pool_r02.ncu-rep --page raw --csv > gpurun_out/prof_c5pool_r02_raw.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tcsearch --launch-skip 5 --launch-count 1 \
    -f -o gpurun_out/prof_b4_r02 python scripts/one_encode.py C3 1 > gpurun_out/ncu_b4_r02.log 2>&1
ls -la gpurun_out gpurun_out/r02
