# run_variants.sh name... : gemm_bench on each variant lib
for n in "$@"; do
  echo "== $n"
  MOBI_LIB_PATH=$PWD/vlib/$n/libmobi_b200.so GB_QUICK=1 timeout 300 python tools/gemm_bench.py 2>&1 | tail -6
done
