set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.err
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/b_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k regex:RowOpE2 -c 3 -o gpurun_out/prof_sweep $SMALL > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
ls -la gpurun_out
