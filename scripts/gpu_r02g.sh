# E16 kernel split + device-setup AINV: tests, bench A/B, AINV line (1 GPU)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py tests/test_gpu_ainv.py -x -q > gpurun_out/g_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/g_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity"
for v in 1 0 1 0; do
  PSC_COL16=$v timeout 600 $B > gpurun_out/g_bench_$v.json 2> gpurun_out/g_bench_$v.err; echo "col16=$v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/g_bench_$v.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'], d['clocks']['reasons'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,1): print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'])"
done
timeout 900 $B --smoother ainv > gpurun_out/g_bench_ainv.json 2> gpurun_out/g_bench_ainv.err; echo ainv_rc=$?
tail -2 gpurun_out/g_bench_ainv.err
python -c "
import json; d=json.load(open('gpurun_out/g_bench_ainv.json')); print(d['metric'], round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['config']['setup_s'], d['roofline'])"
