# round-2 profiles: bench sweep (JSON lines), launch list of the default bench, ncu --set full of the
# hot kernels (prefill GEMM / router at the headline shape, the MLP T=8192 GEMM, the decode pair)
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=gpurun_out/sweep_r2.jsonl; : > $S
run() { timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 100 "$@" 2>/dev/null | tail -1 >> $S; }
for b in 2.0 2.5 3.0 3.5 4.0; do run --target-bits $b; done
run --out 1024 --in 4096
run --out 14336 --in 4096 --tokens 8192 --steps 30
run --out 4096 --in 14336 --tokens 8192 --steps 30
for T in 64 128 512; do run --tokens $T; done
for T in 1 2 4 8 16 32; do run --tokens $T; done
run --out 1024 --in 4096 --tokens 1
run --out 14336 --in 4096 --tokens 1
run --out 4096 --in 14336 --tokens 1
run --hidden 256
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 6 -c 1 -o gpurun_out/r2_gemm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_tc2 -s 6 -c 1 -o gpurun_out/r2_router python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 3 -c 1 -o gpurun_out/r2_gemm_mlp python bench.py --out 14336 --in 4096 --tokens 8192 --steps 2 --warmup 3 --ring 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router_dec|decode_planes" -s 8 -c 2 -o gpurun_out/r2_decode python bench.py --tokens 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
