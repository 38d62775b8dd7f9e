# round-2 final validation (after the calibration steps and the shared workspace): full GPU suite, smoke, C++ drop-in,
# headline bench + reference arm, launch list of the default bench
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m pytest tests -q -m gpu > gpurun_out/g_pytest.log 2>&1; tail -3 gpurun_out/g_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; tail -2 gpurun_out/g_smoke.log
timeout 600 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -1 gpurun_out/g_bench.json | cut -c1-200
tail -1 gpurun_out/g_bench_ref.json | cut -c1-200
