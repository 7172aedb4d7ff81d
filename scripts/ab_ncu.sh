#!/bin/bash
# GPU box: ncu durations of selected kernels (regex $1) in one C3 encode, default build and abvar/*.so
for so in default abvar/*.so; do
  if [ "$so" = default ]; then unset FIC_SO; else export FIC_SO=$PWD/$so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"$1" python scripts/one_encode.py C3 1 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; out=[dict(zip(h,r)) for r in rows[1:]]
out=out[len(out)//2:]
print('$so', ' '.join('%s=%.1fus' % (d['Kernel Name'].split('(')[0].split()[-1][:18], float(d['Metric Value'].replace(',',''))/1000) for d in out))"
done
