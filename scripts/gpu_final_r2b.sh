# round-2 end profiles (after the decode / gather changes): headline bench + reference arm, the shape /
# budget / decode sweep, the launch list of the default bench, ncu --set full of the gate/up decode pair
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
S=gpurun_out/sweep_final.jsonl; : > $S
run() { timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 100 "$@" 2>/dev/null | tail -1 >> $S; }
for b in 2.0 2.5 3.0 3.5 4.0; do run --target-bits $b; done
run --out 1024 --in 4096
run --out 14336 --in 4096 --tokens 8192 --steps 30
run --out 4096 --in 14336 --tokens 8192 --steps 30
for T in 64 128 512; do run --tokens $T; done
for T in 1 2 4 8 16 32; do run --tokens $T; done
for s in "1024 4096" "14336 4096" "4096 14336"; do set -- $s; for T in 1 4 16; do run --out $1 --in $2 --tokens $T; done; done
run --hidden 256
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"router_dec|decode_planes" -s 8 -c 2 -o gpurun_out/r2_decode_gu python bench.py --out 14336 --in 4096 --tokens 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
tail -1 gpurun_out/bench_final.json | cut -c1-300
tail -1 gpurun_out/bench_ref_final.json | cut -c1-300
wc -l $S
