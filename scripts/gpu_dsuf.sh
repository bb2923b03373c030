#!/bin/bash
# dense suffix operator: 1-GPU parity + A/B + launch list
mkdir -p gpurun_out
T=${1:-dsuf}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vbm.py -q -x -m "gpu and not slow" > gpurun_out/${T}_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/${T}_parity.log
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_$1.json 2> gpurun_out/${T}_bench_$1.err; echo "bench_$1_rc=$?"; }
run on; PSC_DENSE_SUFFIX_ROWS=0 run off; run on2; PSC_DENSE_SUFFIX_ROWS=0 run off2
PSC_DENSE_SUFFIX_ROWS=600 run on600
timeout 600 python bench.py --grid 128 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c2_on.json 2>/dev/null
PSC_DENSE_SUFFIX_ROWS=0 timeout 600 python bench.py --grid 128 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c2_off.json 2>/dev/null
timeout 600 python bench.py --problem jump --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_jump_on.json 2>/dev/null
PSC_DENSE_SUFFIX_ROWS=0 timeout 600 python bench.py --problem jump --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_jump_off.json 2>/dev/null
for f in gpurun_out/${T}_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value']), d['config']['iters'][0], round(d['ms_per_step'],2), d['launches_per_iteration'], d['config']['setup_s'])" 2>/dev/null; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_rc=$?"
