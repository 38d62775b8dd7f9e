# quick: gpu tests, gemm_bench (impl $1), bench default
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
MOBI_IMPL=${1:-0} timeout 300 python tools/gemm_bench.py 2>&1 | tail -12
timeout 300 python bench.py --no-cpu-baseline --steps 100 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
