# quick iteration: gpu tests (subset or all), gemm_bench, bench line summary
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 200 ${TESTS:-} > gpurun_out/it_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/it_tests.log
timeout 300 python tools/gemm_bench.py 2>&1 | tail -12
timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "import json; d=json.load(open('gpurun_out/it_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
