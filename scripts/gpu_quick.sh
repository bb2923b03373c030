# quick perf check (under gpurun): bench + A/B env variant + launch list
TAG=${1:-q}
AB=${2:-PSC_NO_RG_TMA=1}
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$B > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?; tail -2 gpurun_out/${TAG}_bench.err
env $AB $B > gpurun_out/${TAG}_bench_nodia.json 2>/dev/null; echo ab_rc=$?
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
