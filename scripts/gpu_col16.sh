# 16-bit column slices: parity tests, then the bench with and without (1 GPU)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/c16_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/c16_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity"
for v in 1 0 1 0; do
  PSC_COL16=$v timeout 600 $B > gpurun_out/c16_bench_$v.json 2> gpurun_out/c16_bench_$v.err; echo "col16=$v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/c16_bench_$v.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,1) or r['level']==-1: print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'])"
done
