# correctness (gpu tests, bounded) then quick perf (under gpurun)
TAG=${1:-c}
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/${TAG}_gpu_tests.log
bash scripts/gpu_quick.sh $TAG
