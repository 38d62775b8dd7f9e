set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 90 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max,launch__grid_size --clock-control none -s 12 -c 8 --csv --log-file gpurun_out/small_t.csv python bench.py --tokens 1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/small_t.csv')) if len(r)>10]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r)); print(d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
