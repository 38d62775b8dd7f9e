# final-build shape / budget / decode sweep (bench.py lines) for profiles/round2_sweep.*
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
S=gpurun_out/sweep_final3.jsonl; : > $S
run() { timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 100 "$@" 2>/dev/null | tail -1 >> $S; }
for b in 2.0 2.5 3.0 3.5 4.0; do run --target-bits $b; done
run --out 1024 --in 4096
run --out 14336 --in 4096 --tokens 8192 --steps 30
run --out 4096 --in 14336 --tokens 8192 --steps 30
for T in 64 128 512; do run --tokens $T; done
for T in 1 2 4 8 16 32; do run --tokens $T; done
for s in "1024 4096" "14336 4096" "4096 14336"; do set -- $s; for T in 1 4 16; do run --out $1 --in $2 --tokens $T; done; done
run --hidden 256
wc -l $S
