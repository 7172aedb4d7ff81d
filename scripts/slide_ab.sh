for so in default $(ls abvar/*.so); do
  if [ "$so" = default ]; then unset FIC_SO; else export FIC_SO=$PWD/$so; fi
  timeout 300 ncu --clock-control none -k regex:"entropy_slide" --metrics gpu__time_duration.sum --csv python scripts/one_encode.py C3 1 > gpurun_out/sl.csv 2>&1
  python - "$so" <<'PY'
import csv, sys
rows=[r for r in csv.reader(open('gpurun_out/sl.csv')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
print(sys.argv[1], [r[vi] for r in rows[1:]])
PY
done
