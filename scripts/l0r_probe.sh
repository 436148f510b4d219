# slots-6 (level 0 ring-resident) A/B (dev).  usage: bash scripts/l0r_probe.sh OUT
D=gpurun_out/$1; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_cta_shape" > $D/shapes.log 2>&1; tail -3 $D/shapes.log
for rep in 1 2; do
timeout 600 python scripts/perf_probe.py --levels 48 --depths 2,3,4 --shapes 0,65,66,67,68,69,70,71,75 2>&1 | grep -v "^{" >> $D/p64.txt
timeout 600 python scripts/perf_probe.py --levels 48 --dtype f32 --nz 2048 --depths 3,4 --shapes 0,72,73 2>&1 | grep -v "^{" >> $D/p32.txt
timeout 600 python scripts/perf_probe.py --levels 48 --depths 6,8 --shapes 0,74 2>&1 | grep -v "^{" >> $D/p64d.txt
done
cat $D/p64.txt $D/p32.txt $D/p64d.txt
