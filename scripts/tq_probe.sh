# tq_kernel (TMEM z-queue) parity + A/B (dev).  usage: bash scripts/tq_probe.sh OUT "shapes64" "shapes32" [depths64] [depths32] [ksel]
D=gpurun_out/$1; mkdir -p $D
S64=$2; S32=$3; D64=${4:-2,3,4,5,6}; D32=${5:-2,3,4,5,6,8}; K=${6:-every_cta_shape}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > $D/shapes.log 2>&1; tail -5 $D/shapes.log
for rep in 1 2; do
[ -n "$S64" ] && timeout 600 python scripts/perf_probe.py --levels 60 --depths $D64 --shapes $S64 2>&1 | grep -v "^{" >> $D/p64.txt
[ -n "$S32" ] && timeout 600 python scripts/perf_probe.py --levels 60 --dtype f32 --nz 2048 --depths $D32 --shapes $S32 2>&1 | grep -v "^{" >> $D/p32.txt
done
