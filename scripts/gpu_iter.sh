# quick iteration: gpu tests + default bench + per-config bench + one ncu capture of a kernel ($1 regex)
set -x
make -s -C oracle lib/libmobi_oracle.so 2>&1 | tail -1
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
if [ -n "$1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 -o gpurun_out/prof_$1 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
fi
