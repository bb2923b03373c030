# correctness (gpu tests, bounded) then A/B perf (under gpurun): bash scripts/gpu_check.sh TAG [ENV variants...]
TAG=${1:-c}; shift
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/${TAG}_gpu_tests.log
bash scripts/gpu_ab.sh $TAG "$@"
