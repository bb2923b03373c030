# Usage (under gpurun): bash scripts/gpu_profile.sh TAG [KERNEL_REGEX] [COUNT]
# 1) plain run of the small bench command (must exit 0 before ncu)
# 2) launch list of one 256^3 solve (gpu__time_duration per launch)
# 3) ncu --set full of the first COUNT launches of KERNEL_REGEX
TAG=${1:-r01}
KRE=${2:-^l1_sweep$}
CNT=${3:-4}
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$SMALL > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT -o gpurun_out/${TAG}_full $SMALL > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full_rc=$?
ls -la gpurun_out | tail -5
