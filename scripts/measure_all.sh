# Round measurement: every bench line, the reference arm, GPU tests, smoke, ncu launch list + full captures.
# usage (GPU box): bash scripts/measure_all.sh [OUT_DIR]
D=${1:-gpurun_out/r02}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/smi.txt
timeout 400 python bench.py > $D/bench_c3.json 2> $D/bench_c3.err
timeout 400 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
for T in 1 2 3 8; do timeout 300 python bench.py --depth $T --no-cpu > $D/bench_c3_T$T.json 2> $D/bench_c3_T$T.err; done
for W in c2 c4 c5w c5s; do timeout 400 python bench.py --workload $W --no-cpu > $D/bench_$W.json 2> $D/bench_$W.err; done
for W in c5w; do for T in 1 8; do timeout 400 python bench.py --workload $W --depth $T --no-cpu > $D/bench_${W}_T$T.json 2> $D/bench_${W}_T$T.err; done; done
for W in c2 c4; do timeout 400 python bench.py --workload $W --depth 8 --no-cpu > $D/bench_${W}_T8.json 2> $D/bench_${W}_T8.err; done
for T in 2 4; do timeout 400 python bench.py --storage compressed --depth $T --no-cpu > $D/bench_c3_compressed_T$T.json 2> $D/bench_c3_compressed_T$T.err; done
timeout 900 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $D/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tb_kernel --launch-skip 2 -c 1 -o $D/ncu_full_c3_T4 python scripts/one_pass.py --n 1024 --depth 4 --passes 3 > $D/ncu_full_c3_T4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tb_kernel --launch-skip 2 -c 1 -o $D/ncu_full_c4_T4 python scripts/one_pass.py --n 1024 --nz 2048 --dtype f32 --depth 4 --passes 3 > $D/ncu_full_c4_T4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tb_kernel --launch-skip 2 -c 1 -o $D/ncu_full_c3_T2 python scripts/one_pass.py --n 1024 --depth 2 --passes 3 > $D/ncu_full_c3_T2.log 2>&1
