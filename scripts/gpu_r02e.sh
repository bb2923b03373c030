# two-step Galerkin + 16-bit column slices: tests, setup timings, bench A/B (1 GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py -x -q > gpurun_out/e_setup_tests.log 2>&1; echo setup_tests_rc=$?
tail -2 gpurun_out/e_setup_tests.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/e_parity_tests.log 2>&1; echo parity_tests_rc=$?
tail -2 gpurun_out/e_parity_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity"
for v in 1 0 1 0; do
  PSC_AMG_VERBOSE=1 PSC_COL16=$v timeout 600 $B > gpurun_out/e_bench_$v.json 2> gpurun_out/e_bench_$v.err; echo "col16=$v rc=$?"
  grep psc_amg gpurun_out/e_bench_$v.err | head -5
  python -c "
import json; d=json.load(open('gpurun_out/e_bench_$v.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'], d['config']['setup_s'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,1,-1): print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'], r['layout_bytes'])"
done
PSC_AMG_VERBOSE=1 timeout 900 python bench.py --problem jump --steps 3 --warmup 3 --no-kernel-table --no-cpu-baseline > gpurun_out/e_jump.json 2> gpurun_out/e_jump.err; echo jump_rc=$?
grep psc_amg gpurun_out/e_jump.err
python -c "import json; d=json.load(open('gpurun_out/e_jump.json')); print(round(d['value'],1), d['config']['iters'][0], d['config']['setup_s'])"
