# Same-box A/B of library builds (dev).
# usage: bash scripts/ab_probe.sh OUT "F64_DEPTHS" "F32_DEPTHS" LIB...   (depths "" = skip)
D=gpurun_out/$1; P64=$2; P32=$3; shift 3
mkdir -p $D
for rep in 1 2; do
  for L in "$@"; do
    echo "== $L rep $rep" >> $D/ab.txt
    [ -n "$P64" ] && SP_LIB_PATH=$L timeout 300 python scripts/perf_probe.py --depths $P64 2>&1 | grep -v "^{" >> $D/ab.txt
    [ -n "$P32" ] && SP_LIB_PATH=$L timeout 300 python scripts/perf_probe.py --dtype f32 --nz 2048 --depths $P32 2>&1 | grep -v "^{" | sed 's/^/f32 /' >> $D/ab.txt
  done
done
python scripts/ab_summary.py $D/ab.txt
