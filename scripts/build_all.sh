#!/bin/bash
# build libfic.so and the trace variant (libfic_trace.so) in parallel
cd "$(dirname "$0")/.."
python paper_1501_04140_b200/build.py > /tmp/b_main.log 2>&1 &
python -c "from paper_1501_04140_b200 import build as b; b.build_variant('paper_1501_04140_b200/libfic_trace.so', defines=['FIC_TC_TRACE'])" > /tmp/b_trace.log 2>&1 &
wait
grep -h " error" /tmp/b_main.log /tmp/b_trace.log | head -20
ls -la paper_1501_04140_b200/*.so
