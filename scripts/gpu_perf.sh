# A/B + launch list under gpurun (1 GPU).  Usage: gpu_perf.sh TAG "ENV_A" "ENV_B" ...
TAG=${1:-ab}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_tests.log | tail -8
i=0
for cfg in "" "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_b$i.json 2> gpurun_out/${TAG}_b$i.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_b$i.json')); print('[$cfg]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], round(d['roofline']['avg_launch_us'],1), round(d['roofline']['frac'],3), d['launches_per_iteration'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
PSC_PROFILE_SOLVE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
python scripts/summarize_launches.py gpurun_out/${TAG}_launches.csv --by-grid 2>&1 | head -40
