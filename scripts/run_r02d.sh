# in-place tq kernels + HOIST-4 A/B (dev).  usage: bash scripts/run_r02d.sh OUT
D=gpurun_out/$1; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_compressed.py tests/test_gpu_fullsize.py -q -x > $D/compressed_tests.log 2>&1; tail -3 $D/compressed_tests.log
timeout 600 python scripts/compressed_probe.py --depths 2,3,4,5,8 --levels 48 --chunk 64 > $D/cprobe64.txt 2>&1
timeout 600 python scripts/compressed_probe.py --depths 3,4 --levels 48 --chunk 128 > $D/cprobe128.txt 2>&1
for rep in 1 2; do timeout 600 python scripts/perf_probe.py --levels 60 --depths 4,5 --shapes 124,129,131,132,118,130,124 2>&1 | grep -v "^{" >> $D/p64.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "every_cta_shape and (129 or 130 or 131 or 132)" > $D/shapes.log 2>&1; tail -2 $D/shapes.log
for T in 3 4; do timeout 400 python bench.py --storage compressed --depth $T --no-cpu > $D/bench_c3_compressed_T$T.json 2> $D/bench_c3_compressed_T$T.err; done
