# full check under gpurun (1 GPU): every GPU test, smoke, bench (device set-up), bench --setup host
TAG=${1:-r02}
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_gpu_tests.log | tail -12
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['config']['setup_s'], round(d['roofline']['frac'],3), d['cpu_baseline'], d['e2e']['value'], d['clocks'])" 2>&1 | tail -3
tail -3 gpurun_out/${TAG}_bench.err
