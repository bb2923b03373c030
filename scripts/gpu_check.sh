# quick check under gpurun (1 GPU): GPU tests (optionally a -k filter), smoke, a short bench line
K=${1:-}
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
if [ -n "$K" ]; then timeout 1500 python -m pytest tests/ -q -m gpu -k "$K" -x > gpurun_out/gpu_tests.log 2>&1;
else timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; fi; echo tests_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['cpu_baseline'], d['e2e']['value'], d['launches_per_iteration'], d['clocks'])"
