# status sweep: gpu tests, default bench, a token/shape sweep (no cpu baseline)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 400 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
: > gpurun_out/sweep.jsonl
for args in "--tokens 1 --graph" "--tokens 16 --graph" "--tokens 64 --graph" "--tokens 512" "--tokens 2048 --target-bits 2" "--tokens 2048 --target-bits 4" \
            "--out 14336 --in 4096 --tokens 1 --graph" "--out 14336 --in 4096 --tokens 64 --graph" "--out 4096 --in 14336 --tokens 1 --graph" "--out 14336 --in 4096 --tokens 8192"; do
  timeout 300 python bench.py $args --no-cpu-baseline --no-e2e --steps 100 2>>gpurun_out/sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['args']='$args'; print(json.dumps(d))" >> gpurun_out/sweep.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/sweep.jsonl'):
    d=json.loads(l); r=d['roofline']
    print(d['args'], '|', round(d['value']), 'tok/s', d['ms_per_step'], 'ms', r['bound'], r['frac'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})
PY
