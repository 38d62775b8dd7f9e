mkdir -p gpurun_out
for T in 1 16; do
  timeout 120 python bench.py --tokens $T --steps 320 --warmup 5 --no-cpu-baseline --no-e2e --graph | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph T=$T', d['value'], 'tok/s', d['ms_per_step'], 'ms', {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
timeout 300 ncu --kernel-name regex:"decode_gemm|router_dec" --set full --cache-control none --clock-control none --import-source on -c 2 -o gpurun_out/dec_t1 python bench.py --tokens 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1
timeout 300 ncu --kernel-name regex:"decode_gemm|router_dec" --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_active.avg --cache-control none --clock-control none -c 6 --csv --log-file gpurun_out/dec_t16.csv python bench.py --tokens 16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1
ncu -i gpurun_out/dec_t1.ncu-rep --page details 2>&1 | grep -E "decode_gemm|router_dec|Duration|DRAM Throughput|Memory Throughput|Registers|Achieved Occupancy|Elapsed Cycles|SM Busy" | head -40
cat gpurun_out/dec_t16.csv | grep -E "gpu__time|dram__bytes" | head
