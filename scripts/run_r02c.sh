# GPU check after the FQ defaults (dev).  usage: bash scripts/run_r02c.sh OUT
D=gpurun_out/$1; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; tail -3 $D/gputests.log
timeout 600 python scripts/perf_probe.py --n 512 --levels 120 --depths 4,8 --shapes 0,35,124,118,127,113,111 2>&1 | grep -v "^{" > $D/p64_c2.txt
timeout 600 python scripts/perf_probe.py --levels 56 --depths 6,7,8 --shapes 0,113 2>&1 | grep -v "^{" > $D/p64_T678.txt
for T in 4 3 5; do timeout 400 python bench.py --depth $T --no-cpu > $D/bench_c3_T$T.json 2> $D/bench_c3_T$T.err; done
for W in c4 c2 c5w; do timeout 400 python bench.py --workload $W --no-cpu > $D/bench_$W.json 2> $D/bench_$W.err; done
