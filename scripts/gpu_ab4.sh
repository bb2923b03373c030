#!/bin/bash
# wavefront with 2048-row items: parity + A/B on one box
mkdir -p gpurun_out
T=${1:-ab4}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" -k "variants" > gpurun_out/${T}_parity.log 2>&1; echo "parity_rc=$?"
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$1.json 2> gpurun_out/${T}_bench_$1.err; echo "bench_$1_rc=$?"; }
run base
PSC_WAVE=1 run wave
PSC_WAVE=1 PSC_WAVE_SLACK=4 run wave_s4
PSC_WAVE=1 PSC_WAVE_SLACK=100 run wave_s100
PSC_WAVE=1 PSC_WAVE_DIRECT=1 run wave_direct
tail -2 gpurun_out/${T}_parity.log
for f in gpurun_out/${T}_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), d['config']['iters'][0], round(d['ms_per_step'],2), round(r['avg_launch_us'],1), round(r['frac'],3), d['launches_per_iteration'])" 2>/dev/null; done
PSC_WAVE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_wave.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_rc=$?"
