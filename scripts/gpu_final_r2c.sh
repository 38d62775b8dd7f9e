# round-2 final validation on the final build: GPU tests, smoke, headline bench + reference arm,
# launch list, ncu --set full of the headline GEMM
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m pytest tests -q -m gpu > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final2.json 2> gpurun_out/bench_ref_final2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 6 -c 1 -o gpurun_out/r2_gemm_final -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out/r2_gemm_final.ncu-rep
tail -1 gpurun_out/bench_final2.json | cut -c1-200
tail -1 gpurun_out/bench_ref_final2.json | cut -c1-200
