# Round evidence (under gpurun, 1 GPU): tests, smoke, full bench line, reference arm,
# launch list, ncu --set full of the dominant kernel.  TAG = round tag.
TAG=${1:-r01}
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/${TAG}_gpu_tests.log
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref_rc=$?
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/${TAG}_plain.log 2>&1 && \
PSC_PROFILE_SOLVE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
PSC_PROFILE_SOLVE=1 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:sell_tma<\(psc::RowOp\)2>' -c 2 -o gpurun_out/${TAG}_l0sweep $SMALL > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full_rc=$?
# the VBM configuration (FCG + coarsest PCG) bench line
python bench.py --vbm --no-cpu-baseline > gpurun_out/${TAG}_bench_vbm.json 2> gpurun_out/${TAG}_bench_vbm.err; echo vbm_rc=$?
