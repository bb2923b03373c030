# parity tests (col16 gate) + exchange microbenchmark (gpurun --gpus 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/f_parity_tests.log 2>&1; echo parity_tests_rc=$?
tail -2 gpurun_out/f_parity_tests.log
bash scripts/gpu_xbench.sh 2
