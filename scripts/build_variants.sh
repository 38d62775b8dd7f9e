# build_variants.sh name1 "EXTRA flags1" name2 "EXTRA flags2" ... -> vlib/<name>/libmobi_b200.so
set -e
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  mkdir -p vlib/$n
  make -s -C paper_2602_20191_b200/csrc OUT=$PWD/vlib/$n/libmobi_b200.so OBJDIR=$PWD/vlib/$n/obj EXTRA="$f" -j8 2>&1 | grep -E "error" || true
  ls -la vlib/$n/libmobi_b200.so
done
