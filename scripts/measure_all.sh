# Round measurement: every bench line, the reference arm, GPU tests, smoke, ncu launch list + full captures.
# usage (GPU box): bash scripts/measure_all.sh [OUT_DIR]
D=${1:-gpurun_out/r02}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 400 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 400 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
for T in 1 2 3 5 8; do timeout 300 python bench.py --depth $T --no-cpu > $D/bench_c3_T$T.json 2> $D/bench_c3_T$T.err; done
for W in c2 c4 c5w c5s; do timeout 400 python bench.py --workload $W --no-cpu > $D/bench_$W.json 2> $D/bench_$W.err; done
for W in c5w; do for T in 1 8; do timeout 400 python bench.py --workload $W --depth $T --no-cpu > $D/bench_${W}_T$T.json 2> $D/bench_${W}_T$T.err; done; done
for W in c2 c4; do timeout 400 python bench.py --workload $W --depth 8 --no-cpu > $D/bench_${W}_T8.json 2> $D/bench_${W}_T8.err; done
for T in 3 4; do timeout 400 python bench.py --storage compressed --depth $T --no-cpu > $D/bench_c3_compressed_T$T.json 2> $D/bench_c3_compressed_T$T.err; done
timeout 900 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $D/ncu_launch.log 2>&1
# full captures go to /tmp on the box (reports of this kernel exceed gpurun's copy-back limit);
# their summaries (details page, raw metrics, instruction mix) come back in $D
mkdir -p /tmp/ncu_full
for C in "c3_T4 --n 1024 --depth 4" "c4_T4 --n 1024 --nz 2048 --dtype f32 --depth 4" "c3_T2 --n 1024 --depth 2" "c3_T3 --n 1024 --depth 3" "c3_T5 --n 1024 --depth 5" "c3_T8 --n 1024 --depth 8"; do
  set -- $C; N=$1; shift
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:t[bq]_kernel --launch-skip 2 -c 1 -o /tmp/ncu_full/$N python scripts/one_pass.py "$@" --passes 3 > $D/ncu_full_$N.log 2>&1
  python scripts/summarize_ncu.py full /tmp/ncu_full/$N.ncu-rep $D/ncu_full_$N >> $D/ncu_full_$N.log 2>&1
  python scripts/ncu_mix2.py /tmp/ncu_full/$N.ncu-rep 12 > $D/step_mix_$N.txt 2>&1
done
