# compute-sanitizer evidence (1 GPU): memcheck, racecheck, synccheck on scripts/sanitize_case.py
TAG=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_case.py > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|ALL OK|FAILED|Invalid|Race|Barrier" gpurun_out/${TAG}_sanitize_${tool}.log | head -5
done
