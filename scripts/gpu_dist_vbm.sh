#!/bin/bash
# multi-GPU (under gpurun --gpus N): dist parity incl. the VBM leg, VBM + PCG bench at N
N=${1:-2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/dvbm${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -15 gpurun_out/dvbm${N}_tests.log | grep -v "^$" | tail -8
for extra in "" "--vbm"; do
  tag=$( [ -z "$extra" ] && echo pcg || echo vbm )
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e $extra > gpurun_out/dvbm${N}_bench_${tag}.json 2> gpurun_out/dvbm${N}_bench_${tag}.err; echo "bench $tag rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/dvbm${N}_bench_${tag}.json').read().strip().splitlines()[-1]); print('$tag', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['halo_path'], d['launches_per_iteration'])"
done
