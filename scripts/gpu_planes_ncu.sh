# ncu --set full of the decode planes kernel (T=$1, default 4), with source-level stalls
mkdir -p gpurun_out
T=${1:-4}
timeout 300 ncu --kernel-name regex:"decode_planes" --set full --clock-control none --import-source on -s 3 -c 1 -o gpurun_out/planes_t$T -f python bench.py --tokens $T --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > gpurun_out/planes_ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/planes_ncu.log
