# GPU check after the tq_kernel defaults (dev).  usage: bash scripts/run_r02b.sh OUT
D=gpurun_out/$1; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; tail -3 $D/gputests.log
timeout 600 python scripts/perf_probe.py --levels 56 --depths 7,8 --shapes 0,76,87,89 2>&1 | grep -v "^{" > $D/p64_T78.txt
timeout 600 python scripts/perf_probe.py --levels 56 --dtype f32 --nz 2048 --depths 7,8 --shapes 0,76,77,81,86,87,89,93 2>&1 | grep -v "^{" > $D/p32_T78.txt
timeout 400 python bench.py --workload c4 --no-cpu > $D/bench_c4.json 2> $D/bench_c4.err
timeout 400 python bench.py --depth 3 --no-cpu > $D/bench_c3_T3.json 2> $D/bench_c3_T3.err
timeout 400 python bench.py --no-cpu > $D/bench_c3.json 2> $D/bench_c3.err
