#!/bin/bash
# exchange/interior overlap on N GPUs: dist parity + A/B
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vbm.py -q -x -m "gpu and not slow" > gpurun_out/ovl${N}_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/ovl${N}_parity.log
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/ovl${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -2 gpurun_out/ovl${N}_tests.log
for v in ovl noovl ovl2 noovl2; do
  case $v in noovl*) E="PSC_NO_OVERLAP=1";; *) E="";; esac
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e > gpurun_out/ovl${N}_$v.json 2> gpurun_out/ovl${N}_$v.err; echo "bench $v rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/ovl${N}_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['launches_per_iteration'])"
done
