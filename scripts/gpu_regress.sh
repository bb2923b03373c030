#!/bin/bash
# same-box A/B: libpsc_a.so (530c55e, before chunk lists) vs current; dense suffix on/off; launch lists
mkdir -p gpurun_out
T=reg
for rep in 1 2; do
for v in a cur cur_nods; do
  case $v in a) L=libpsc_a.so; E="";; cur) L=libpsc.so; E="";; cur_nods) L=libpsc.so; E="PSC_DENSE_SUFFIX_ROWS=0";; esac
  env $E PSC_LIB=$PWD/paper_2406_19754_b200/$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${T}_$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value'],1), round(d['ms_per_step'],2), round(r['avg_launch_us'],1), d['launches_per_iteration'])"
done; done
for v in a cur; do
  case $v in a) L=libpsc_a.so;; cur) L=libpsc.so;; esac
  PSC_LIB=$PWD/paper_2406_19754_b200/$L PSC_PROFILE_SOLVE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_$v rc=$?"
done
