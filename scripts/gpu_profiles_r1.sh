# round-1 profile batch: bench lines, ncu launch list, full captures of the GEMM / router / decode kernels,
# shape sweep, model-stack sweep.  Everything lands in gpurun_out/ (copied to profiles/ afterwards).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/p_gpu.txt
timeout 600 python bench.py > gpurun_out/p_bench_default.json 2> gpurun_out/p_bench_default.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/p_bench_reference.json 2>&1; echo ref rc=$?
: > gpurun_out/p_sweep.jsonl
for args in "--tokens 1" "--tokens 2" "--tokens 4" "--tokens 8" "--tokens 16" "--tokens 32" "--tokens 64" "--tokens 128" "--tokens 512" "--tokens 2048 --target-bits 2" "--tokens 2048 --target-bits 2.5" "--tokens 2048 --target-bits 3.5" "--tokens 2048 --target-bits 4" "--tokens 2048 --hidden 256" \
            "--out 1024 --in 4096 --tokens 2048" "--out 14336 --in 4096 --tokens 1" "--out 14336 --in 4096 --tokens 16" "--out 14336 --in 4096 --tokens 64" "--out 4096 --in 14336 --tokens 1" "--out 4096 --in 14336 --tokens 64" "--out 14336 --in 4096 --tokens 8192" "--out 4096 --in 14336 --tokens 8192"; do
  timeout 300 python bench.py $args --no-cpu-baseline --no-e2e --steps 100 2>>gpurun_out/p_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['args']='$args'; print(json.dumps(d))" >> gpurun_out/p_sweep.jsonl
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 30 --csv --log-file gpurun_out/p_launches.csv python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 3 -c 1 -o gpurun_out/p_gemm python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo gemm rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_tc2 -s 3 -c 1 -o gpurun_out/p_router python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo router rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_planes|router_dec" -s 4 -c 2 -o gpurun_out/p_decode python bench.py --tokens 1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo decode rc=$?
timeout 900 python tools/stack_sweep.py --blocks 32 --tokens 2048 --steps 5 > gpurun_out/p_stack_sweep.jsonl 2> gpurun_out/p_stack_sweep.err; echo stack rc=$?
