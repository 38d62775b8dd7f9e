# bench_variants.sh name... : default bench line (GEMM/router/gather per-kernel times) per variant lib
for n in "$@"; do
  MOBI_LIB_PATH=$PWD/vlib/$n/libmobi_b200.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['ms_per_step'], d['roofline']['frac'], {k:v['ms_per_launch'] for k,v in d['kernels'].items()})"
done
