#!/bin/bash
# wavefront pass: L2 bandwidth probe, parity with PSC_WAVE=1, A/B bench on one box
mkdir -p gpurun_out
T=${1:-wave}
./scripts/bin/l2bw > gpurun_out/${T}_l2bw.txt 2>&1; echo "l2bw_rc=$?"
PSC_WAVE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" -k "vcycle or pcg" > gpurun_out/${T}_parity.log 2>&1; echo "wave_parity_rc=$?"
timeout 1200 python -m pytest tests/test_gpu_vbm.py -q > gpurun_out/${T}_vbm_tests.log 2>&1; echo "vbm_tests_rc=$?"
for v in 0 1; do
  if [ $v = 1 ]; then export PSC_WAVE=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_w$v.json 2> gpurun_out/${T}_bench_w$v.err; echo "bench_w${v}_rc=$?"
done
PSC_WAVE=1 PSC_WAVE_SLACK=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_w1_s0.json 2>/dev/null; echo "slack0_rc=$?"
PSC_WAVE=1 PSC_WAVE_SLACK=300 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_w1_s300.json 2>/dev/null; echo "slack300_rc=$?"
cat gpurun_out/${T}_l2bw.txt
tail -2 gpurun_out/${T}_parity.log gpurun_out/${T}_vbm_tests.log
