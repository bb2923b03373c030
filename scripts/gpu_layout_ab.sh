#!/bin/bash
# layout A/B on one box: row-group threshold (levels 1-2 as row groups), L2 keep budget
mkdir -p gpurun_out
T=${1:-lay}
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$1.json 2> gpurun_out/${T}_bench_$1.err; echo "bench_$1_rc=$?"; }
run base
PSC_RG_MIN=64 run rg64
PSC_RG_MIN=24 run rg24
PSC_RG_MIN=64 PSC_RG_DIV=2 run rg64d2
PSC_RG_MIN=24 PSC_RG_DIV=4 run rg24d4
run base2
for f in gpurun_out/${T}_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), d['config']['iters'][0], round(d['ms_per_step'],2), round(r['avg_launch_us'],1), round(r['frac'],3), d['launches_per_iteration'])" 2>/dev/null; done
PSC_RG_MIN=64 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_rg64.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_rc=$?"
