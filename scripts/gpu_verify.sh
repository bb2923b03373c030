#!/bin/bash
# after removing the chunk lists: same-box A/B vs libpsc_a.so, 1-GPU parity
mkdir -p gpurun_out
for rep in 1 2; do for L in libpsc_a.so libpsc.so; do
  PSC_LIB=$PWD/paper_2406_19754_b200/$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ver_$L.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ver_$L.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$L', round(d['value'],1), round(d['ms_per_step'],2), round(r['avg_launch_us'],1), d['launches_per_iteration'])"
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vbm.py -q -x -m "gpu and not slow" > gpurun_out/ver_parity.log 2>&1; echo parity_rc=$?; tail -1 gpurun_out/ver_parity.log
