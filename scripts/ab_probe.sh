# Same-box A/B of library builds (dev).  usage: bash scripts/ab_probe.sh OUT LIB_A LIB_B [f64 depths] [f32 depths]
D=gpurun_out/$1; A=$2; B=$3; P64=${4:-2,3,4}; P32=${5:-2,3,4}
mkdir -p $D
for rep in 1 2; do
  for L in $A $B; do
    echo "== $L rep $rep" >> $D/ab.txt
    SP_LIB_PATH=$L timeout 300 python scripts/perf_probe.py --depths $P64 2>&1 | grep -v "^{" >> $D/ab.txt
    SP_LIB_PATH=$L timeout 300 python scripts/perf_probe.py --dtype f32 --nz 2048 --depths $P32 2>&1 | grep -v "^{" | sed 's/^/f32 /' >> $D/ab.txt
  done
done
cat $D/ab.txt
