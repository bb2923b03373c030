#!/bin/bash
# deferred fused exchange on N GPUs: parity + A/B; 1-GPU library A/B (prev vs current)
N=${1:-2}
mkdir -p gpurun_out
for rep in 1 2; do for lib in libpsc_prev.so libpsc.so; do
  PSC_LIB=$PWD/paper_2406_19754_b200/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/def_$lib.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/def_$lib.json').read().strip().splitlines()[-1]); print('1gpu [$lib]', round(d['value'],1), round(d['ms_per_step'],2))"
done; done
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/def${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -2 gpurun_out/def${N}_tests.log
for v in base defer base2 defer2; do
  case $v in defer*) E="PSC_DEFER_EXCHANGE=1";; *) E="";; esac
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e > gpurun_out/def${N}_$v.json 2> gpurun_out/def${N}_$v.err; echo "bench $v rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/def${N}_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['launches_per_iteration'])"
done
