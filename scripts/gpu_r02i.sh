# AINV: own-x prefetch for square Spmv / PAdd (1 GPU): tests + AINV bench A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ainv.py tests/test_gpu_setup.py -x -q > gpurun_out/i_tests.log 2>&1; echo tests_rc=$?
tail -1 gpurun_out/i_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --smoother ainv"
for v in 0 1 0; do
  PSC_NO_XPRE=$v timeout 900 $B > gpurun_out/i_ainv_$v.json 2> gpurun_out/i_ainv_$v.err; echo "no_xpre=$v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/i_ainv_$v.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,): print('  ', r['kernel'], r['level'], r['calls_per_iter'], r['us_per_call'], r['layout_frac'])"
done
