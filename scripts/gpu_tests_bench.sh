# tests + smoke + bench + launch list (under gpurun)
TAG=${1:-r01}
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/${TAG}_gpu_tests.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
tail -2 gpurun_out/${TAG}_bench.err
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
# A/B: same bench without DIA slices
PSC_NO_DIA=1 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_nodia.json 2>/dev/null; echo nodia_rc=$?
