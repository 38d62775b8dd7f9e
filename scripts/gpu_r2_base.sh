# round-2 baseline: gpu tests, gemm_bench (all distributions), traced tc2 at the bench shape, bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/r2_gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_gpu_tests.log
timeout 300 python tools/gemm_bench.py > gpurun_out/r2_gemm_bench.txt 2>&1; tail -14 gpurun_out/r2_gemm_bench.txt
MOBI_TRACE_IMPL=4 timeout 200 python tools/gemm_trace.py > gpurun_out/r2_gemm_trace.txt 2>&1; tail -50 gpurun_out/r2_gemm_trace.txt
timeout 300 python bench.py --steps 100 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 600 gpurun_out/r2_bench.json
