# 2-GPU check of the multi-rank AINV leg and the warp-stage Galerkin (gpurun --gpus 2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py tests/test_gpu_ainv.py -x -q > gpurun_out/as_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/as_tests.log
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -k "two_gpu_parity or jump" > gpurun_out/as_dist.log 2>&1; echo dist_rc=$?
tail -2 gpurun_out/as_dist.log
PSC_AMG_VERBOSE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-kernel-table --no-parity > gpurun_out/as_bench.json 2> gpurun_out/as_bench.err; echo bench_rc=$?
grep psc_amg gpurun_out/as_bench.err
python -c "import json; d=json.load(open('gpurun_out/as_bench.json')); print(round(d['value'],1), d['config']['setup_s'])"
PSC_AMG_VERBOSE=1 timeout 900 python bench.py --problem jump --steps 3 --warmup 3 --no-kernel-table --no-cpu-baseline > gpurun_out/as_jump.json 2> gpurun_out/as_jump.err; echo jump_rc=$?
grep psc_amg gpurun_out/as_jump.err; tail -3 gpurun_out/as_jump.err
python -c "import json; d=json.load(open('gpurun_out/as_jump.json')); print(round(d['value'],1), d['config']['iters'][0], d['config']['setup_s'])"
