#!/bin/bash
N=${1:-2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/dsuf${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -1 gpurun_out/dsuf${N}_tests.log
for v in on off; do
  case $v in off) E="PSC_DENSE_SUFFIX_ROWS=0";; *) E="";; esac
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e > gpurun_out/dsuf${N}_$v.json 2> gpurun_out/dsuf${N}_$v.err; echo "bench $v rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/dsuf${N}_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['launches_per_iteration'], d['config']['setup_s'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e --vbm > gpurun_out/dsuf${N}_vbm.json 2> gpurun_out/dsuf${N}_vbm.err; echo "bench vbm rc=$?"
