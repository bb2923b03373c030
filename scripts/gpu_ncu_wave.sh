#!/bin/bash
# A/B of the wave after the own-x prefetch, then one ncu --set full capture of a level-0 sell_wave launch
mkdir -p gpurun_out
T=${1:-ncuwave}
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$1.json 2> gpurun_out/${T}_bench_$1.err; echo "bench_$1_rc=$?"; }
run w0
PSC_WAVE=1 run w1
PSC_WAVE=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^sell_wave$ -s 1 -c 1 -o gpurun_out/${T} python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu_rc=$?"
for f in gpurun_out/${T}_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), d['config']['iters'][0], round(d['ms_per_step'],2), round(r['avg_launch_us'],1), round(r['frac'],3), d['launches_per_iteration'])" 2>/dev/null; done
PSC_WAVE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_rc=$?"
