# launch list for an arbitrary bench argument string (under gpurun): bash scripts/gpu_list2.sh TAG "ARGS" ["ENV"]
TAG=$1; ARGS=$2; CFG=$3
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e $ARGS"
env $CFG $SMALL > gpurun_out/${TAG}_plain.log 2>&1 || { echo plain failed; tail gpurun_out/${TAG}_plain.log; exit 1; }
env $CFG ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
