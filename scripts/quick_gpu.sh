# Quick GPU check (dev): GPU tests + kernel-only probes.  usage: bash scripts/quick_gpu.sh OUT [probe args...]
D=gpurun_out/$1; shift
mkdir -p $D
timeout 600 python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; tail -2 $D/gputests.log
timeout 300 python scripts/perf_probe.py --depths 1,2,3,4,6,8 > $D/probe64.txt 2>&1; grep -v "^{" $D/probe64.txt
timeout 300 python scripts/perf_probe.py --dtype f32 --nz 2048 --depths 1,2,3,4,8 > $D/probe32.txt 2>&1; grep -v "^{" $D/probe32.txt
