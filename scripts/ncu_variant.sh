# ncu --set full of one pass of a given variant; raw CSV + details come back (dev).
# usage: bash scripts/ncu_variant.sh OUT NAME "one_pass args"
D=gpurun_out/$1; N=$2; shift 2
mkdir -p $D /tmp/ncu_full
timeout 600 ncu --set full --import-source on --clock-control none -k regex:t[bq]_kernel --launch-skip 2 -c 1 -f -o /tmp/ncu_full/$N python scripts/one_pass.py $@ --passes 3 > $D/ncu_$N.log 2>&1
ncu -i /tmp/ncu_full/$N.ncu-rep --page raw --csv > $D/${N}_rawfull.csv 2>/dev/null
ncu -i /tmp/ncu_full/$N.ncu-rep --page details > $D/${N}_details.txt 2>/dev/null
python scripts/ncu_mix2.py /tmp/ncu_full/$N.ncu-rep 30 > $D/${N}_mix.txt 2>&1
