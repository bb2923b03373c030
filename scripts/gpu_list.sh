# launch list for one env config (under gpurun): bash scripts/gpu_list.sh TAG "ENV"
TAG=$1; CFG=$2
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
env $CFG $SMALL > gpurun_out/${TAG}_plain.log 2>&1 || { echo plain failed; exit 1; }
env $CFG ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
