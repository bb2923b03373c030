#!/bin/bash
# NEXT-2 (VBM: FCG + coarsest PCG) parity + bench on one B200
mkdir -p gpurun_out
T=${1:-vbm}
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_vbm.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo "vbm_tests_rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" > gpurun_out/${T}_parity.log 2>&1; echo "parity_rc=$?"
timeout 600 python bench.py --vbm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_vbm.json 2> gpurun_out/${T}_bench_vbm.err; echo "bench_vbm_rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_pcg.json 2> gpurun_out/${T}_bench_pcg.err; echo "bench_pcg_rc=$?"
timeout 600 python bench.py --vbm --problem jump --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_vbm_jump.json 2> gpurun_out/${T}_bench_vbm_jump.err; echo "bench_vbm_jump_rc=$?"
tail -3 gpurun_out/${T}_tests.log gpurun_out/${T}_parity.log
