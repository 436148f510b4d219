# Round measurement: every bench line, the reference arm, GPU tests, smoke, ncu launch list.
# usage (GPU box): bash scripts/measure_all.sh [OUT_DIR]
D=${1:-gpurun_out/r01c}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 300 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 300 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
for T in 1 3 4 8; do timeout 300 python bench.py --depth $T --no-cpu > $D/bench_c3_T$T.json 2> $D/bench_c3_T$T.err; done
for W in c2 c4 c5w; do timeout 400 python bench.py --workload $W --no-cpu > $D/bench_$W.json 2> $D/bench_$W.err; done
for W in c2 c4; do timeout 400 python bench.py --workload $W --depth 8 --no-cpu > $D/bench_${W}_T8.json 2> $D/bench_${W}_T8.err; done
for T in 2 3; do timeout 400 python bench.py --storage compressed --depth $T --no-cpu > $D/bench_c3_compressed_T$T.json 2> $D/bench_c3_compressed_T$T.err; done
timeout 900 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu > $D/ncu_launch.log 2>&1
