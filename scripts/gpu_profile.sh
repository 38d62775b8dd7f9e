# profiles for the current kernels: launch list of one bench step sequence + full capture of GEMM and router
set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc_kernel -s 3 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo gemm rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router_tc_kernel -s 3 -c 1 -o gpurun_out/prof_router python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --ring 1 > /dev/null 2>&1; echo router rc=$?
