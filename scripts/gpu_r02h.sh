# dinv2 staged for the Spmv epilogue (R0 / AINV Z^T): tests + bench default and AINV (1 GPU)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ainv.py tests/test_gpu_variable_v.py tests/test_gpu_vbm.py -x -q > gpurun_out/h_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/h_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity"
for k in 1 2; do
  timeout 600 $B > gpurun_out/h_bench_$k.json 2> gpurun_out/h_bench_$k.err; echo "bench rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/h_bench_$k.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in d['kernel_table']['rows']:
    if 'Spmv' in r['kernel'] or 'PAdd' in r['kernel']: print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'])"
done
timeout 900 $B --smoother ainv > gpurun_out/h_bench_ainv.json 2> gpurun_out/h_bench_ainv.err; echo ainv_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/h_bench_ainv.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,): print('  ', r['kernel'], r['level'], r['calls_per_iter'], r['us_per_call'], r['layout_frac'])"
