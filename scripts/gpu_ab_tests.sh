# parity tests, then a same-box A/B (gpu_ab.sh).  Usage: gpu_ab_tests.sh TAG "ENV_A" "ENV_B" [reps]
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ainv.py tests/test_gpu_vbm.py -x -q > gpurun_out/$1_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/$1_tests.log
bash scripts/gpu_ab.sh "$@"
