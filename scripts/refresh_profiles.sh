#!/bin/bash
# GPU-box: bench lines (C3 full, C4, C5), the ncu launch list of the C3 bench and one
# `ncu --set full` capture of the search kernels of one C3 encode, all under gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1
timeout 600 python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tcsearch|b2win" --launch-skip 4 \
    --launch-count 4 -f -o gpurun_out/prof_full python scripts/one_encode.py C3 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/bench_full.log | cut -c1-300
