# more FQ A/B (dev).  usage: bash scripts/run_r02f.sh OUT
D=gpurun_out/$1; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_cta_shape and (133 or 134 or 135 or 136 or 137 or 138 or 139 or 140)" > $D/shapes.log 2>&1; tail -2 $D/shapes.log
for rep in 1 2; do
timeout 600 python scripts/perf_probe.py --levels 60 --depths 4 --shapes 131,131,133,134,140,131 2>&1 | grep -v "^{" >> $D/p64.txt
timeout 600 python scripts/perf_probe.py --levels 60 --depths 5 --shapes 111,111,140,127 2>&1 | grep -v "^{" >> $D/p64_T5.txt
timeout 600 python scripts/perf_probe.py --levels 60 --dtype f32 --nz 2048 --depths 4,5 --shapes 93,93,135,136,137,138,139,126 2>&1 | grep -v "^{" >> $D/p32.txt
done
for C in 2 3 4 5 6 8; do echo "chunks $C" >> $D/chunks.txt; timeout 300 python scripts/perf_probe.py --levels 60 --depths 4 --chunks $C 2>&1 | grep -v "^{" >> $D/chunks.txt; done
