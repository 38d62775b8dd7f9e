mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -15
for T in 1 4 16 32; do
  timeout 120 python bench.py --tokens $T --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --graph | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph T=$T', d['value'], 'tok/s', d['ms_per_step'], 'ms', {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
  timeout 120 python bench.py --tokens $T --steps 300 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager T=$T', d['value'], 'tok/s', d['ms_per_step'], 'ms')"
done
timeout 120 python bench.py --tokens 1 --out 14336 --steps 300 --warmup 5 --no-cpu-baseline --no-e2e --graph | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gate/up graph T=1', d['value'], d['ms_per_step'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('T=2048', d['value'], d['ms_per_step'])"
