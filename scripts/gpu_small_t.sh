mkdir -p gpurun_out
for T in 1 64; do
timeout 300 ncu --kernel-name regex:"gemm_tc|router_tc|router_reduce|bucket_k|gather_k|splitk_red" --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_elapsed.max,launch__grid_size,dram__bytes_read.sum --clock-control none -c 12 --csv --log-file gpurun_out/small_t$T.csv python bench.py --tokens $T --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > gpurun_out/small_t$T.log 2>&1
python - $T <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/small_t{sys.argv[1]}.csv')) if len(r)>10]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r)); print(d['ID'], d['Kernel Name'][:30], d['Metric Name'], d['Metric Value'])
PY
done
