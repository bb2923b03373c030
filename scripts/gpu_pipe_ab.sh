#!/bin/bash
# library A/B on one box: default vs software-pipelined ELL batches
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libpsc.so libpsc_pipe.so; do
  PSC_LIB=$PWD/paper_2406_19754_b200/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pipe_$lib.json 2>gpurun_out/pipe_$lib.err || { echo "FAIL $lib"; tail -3 gpurun_out/pipe_$lib.err; continue; }
  python -c "import json; d=json.loads(open('gpurun_out/pipe_$lib.json').read().strip().splitlines()[-1]); print('[$lib]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0])"
done
done
PSC_LIB=$PWD/paper_2406_19754_b200/libpsc_pipe.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pipe_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list_rc=$?"
