# round-2 re-entry validation of the last GEMM barrier change: GPU tests, smoke, sanitizer (synccheck /
# racecheck), headline bench + reference arm, launch list, ncu --set full of the headline GEMM
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m pytest tests -q -m gpu > gpurun_out/d_pytest.log 2>&1; tail -3 gpurun_out/d_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; tail -2 gpurun_out/d_smoke.log
timeout 600 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/d_bench_ref.json 2> gpurun_out/d_bench_ref.err
for t in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_paths.py > gpurun_out/d_$t.log 2>&1; tail -2 gpurun_out/d_$t.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 6 -c 1 -o gpurun_out/d_gemm -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/d_gemm.ncu-rep
tail -1 gpurun_out/d_bench.json | cut -c1-200
tail -1 gpurun_out/d_bench_ref.json | cut -c1-200
