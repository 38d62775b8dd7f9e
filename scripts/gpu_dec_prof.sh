mkdir -p gpurun_out
for T in 1 16; do
timeout 300 ncu --kernel-name regex:"decode_gemm|router_dec" --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_active.avg,launch__grid_size --clock-control none -c 8 --csv --log-file gpurun_out/dec_t$T.csv python bench.py --tokens $T --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1
python - $T <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(f'gpurun_out/dec_t{sys.argv[1]}.csv')) if len(r)>10]
hdr=rows[0]
for r in rows[1:]:
    d=dict(zip(hdr,r)); print('T',sys.argv[1], d['ID'], d['Kernel Name'][:30], d['Metric Name'], d['Metric Value'])
PY
done
timeout 300 ncu --kernel-name regex:"decode_gemm|router_dec" --set full --clock-control none --import-source on -s 2 -c 2 -o gpurun_out/dec_full python bench.py --tokens 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo full rc=$?
timeout 300 ncu --kernel-name regex:"router_tc" --set full --clock-control none --import-source on -s 2 -c 1 -o gpurun_out/router_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo rfull rc=$?
MOBI_TRACE_IMPL=2 timeout 120 python tools/gemm_trace.py > gpurun_out/trace2.txt 2>&1; echo trace rc=$?; cat gpurun_out/trace2.txt | head -60
MOBI_IMPL=0 timeout 300 python tools/gemm_bench.py > gpurun_out/gb0.txt 2>&1; cat gpurun_out/gb0.txt
MOBI_IMPL=3 timeout 300 python tools/gemm_bench.py > gpurun_out/gb3.txt 2>&1; cat gpurun_out/gb3.txt
