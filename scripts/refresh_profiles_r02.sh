#!/bin/bash
# GPU box, round 2: bench lines (C3 default, C4, C5), the ncu launch list of the C3 bench, and
# `ncu --set full` captures of every kernel of one C3 encode and of the C5 pool kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py > gpurun_out/bench_r02.log 2>&1
timeout 600 python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/bench_c4_r02.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r02.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r02.log 2>&1
# one warm-up encode (~57 launches) skipped, then every kernel of one encode
timeout 1200 ncu --set full --import-source on --clock-control none --launch-skip 60 --launch-count 70 \
    -f -o gpurun_out/prof_c3_r02 python scripts/one_encode.py C3 1 > gpurun_out/ncu_c3_r02.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"entropy|pool|select_chain|t2f" --launch-skip 14 --launch-count 14 \
    -f -o gpurun_out/prof_c5pool_r02 python scripts/one_encode.py C5 1 > gpurun_out/ncu_c5pool_r02.log 2>&1
tail -c 400 gpurun_out/bench_r02.log
