#!/bin/bash
# GPU box, round 2: bench lines (C3 default, C4, C5), the ncu launch list of the C3 bench, and
# `ncu --set full` captures of every kernel of one C3 encode and of the C5 pool kernels (exported
# to CSV on the box; the reports themselves stay there).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py > gpurun_out/bench_r02.log 2>&1
timeout 600 python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/bench_c4_r02.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r02.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r02.log 2>&1
mkdir -p /tmp/reps
timeout 1200 ncu --set full --clock-control none --launch-skip 60 --launch-count 70 \
    -f -o /tmp/reps/prof_c3_r02 python scripts/one_encode.py C3 1 > gpurun_out/ncu_c3_r02.log 2>&1
ncu -i /tmp/reps/prof_c3_r02.ncu-rep --page raw --csv > gpurun_out/prof_c3_r02_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"entropy|pool|select_chain|t2f" --launch-skip 14 --launch-count 14 \
    -f -o /tmp/reps/prof_c5pool_r02 python scripts/one_encode.py C5 1 > gpurun_out/ncu_c5pool_r02.log 2>&1
ncu -i /tmp/reps/prof_c5pool_r02.ncu-rep --page raw --csv > gpurun_out/prof_c5pool_r02_raw.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tcsearch --launch-skip 5 --launch-count 1 \
    -f -o gpurun_out/prof_b4_r02 python scripts/one_encode.py C3 1 > gpurun_out/ncu_b4_r02.log 2>&1
ls -la gpurun_out | head -40
tail -c 400 gpurun_out/bench_r02.log
