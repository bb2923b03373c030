# bounds-checked build (device traps on out-of-range gathers / ring overflows) under the
# GPU parity tests; compute-sanitizer is closed on this pool
TAG=${1:-r02}
mkdir -p gpurun_out
PSC_LIB=$PWD/paper_2406_19754_b200/libpsc_checked.so timeout 2400 python -m pytest tests/ -q -m gpu -x > gpurun_out/${TAG}_checked_tests.log 2>&1; echo checked_rc=$?
tail -3 gpurun_out/${TAG}_checked_tests.log
