#!/bin/bash
# GPU box, round 2: every committed result line (gpurun_out/r02/*): the C3 headline bench, the C3
# t x s-mode matrix and the two other large-s modes, C4, C5 (plain and through fic_encode_nccl on
# a one-rank communicator), C5 with serialised pools, the paper protocols, and the launch list.
set -x
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02/build.log 2>&1 || exit 1
timeout 600 python bench.py > gpurun_out/r02/bench_c3.json 2> gpurun_out/r02/bench_c3.err
for mode in predefined grid; do for t in 4 8 12; do
  timeout 600 python bench.py --s-mode $mode --t $t --steps 30 > gpurun_out/r02/c3_${mode}_t${t}.json 2>/dev/null
done; done
for mode in sampled10 closed5; do
  timeout 600 python bench.py --s-mode $mode --steps 30 > gpurun_out/r02/c3_${mode}_t8.json 2>/dev/null
done
timeout 600 python bench.py --topk 256 --steps 30 > gpurun_out/r02/c3_top256.json 2>/dev/null
timeout 600 python bench.py --config C4 --steps 10 --no-cpu-baseline > gpurun_out/r02/bench_c4.json 2>/dev/null
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_c5.json 2>/dev/null
timeout 900 python bench.py --config C5 --nccl --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/bench_c5_nccl1rank.json 2>/dev/null
timeout 900 python bench.py --config C5 --serial-pools --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r02/bench_c5_serial_pools.json 2>/dev/null
timeout 600 python bench.py --nccl --steps 30 --no-cpu-baseline > gpurun_out/r02/bench_c3_nccl1rank.json 2>/dev/null
timeout 600 python scripts/paper_protocols.py > gpurun_out/r02/paper_protocols.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/r02
