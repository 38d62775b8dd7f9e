set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nproc; free -g | head -2
make -s -C oracle lib/libmobi_oracle.so 2>&1 | tail -1
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; cat gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
for T in 16 128 512; do timeout 300 python bench.py --tokens $T --no-cpu-baseline --steps 200 >> gpurun_out/bench_T.json 2>>gpurun_out/bench_T.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc -s 2 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?; tail -3 gpurun_out/ncu_full.log
