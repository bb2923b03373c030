# fused-push A/B on N GPUs: parity tests with PSC_PUSH=1, then bench default vs PSC_PUSH=1 (twice each)
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "PUSH or two_gpu_parity or four_gpu" > gpurun_out/push${N}_tests.log 2>&1; echo tests_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/push${N}_tests.log | tail -6
for c in "" PSC_PUSH=1 "" PSC_PUSH=1; do
env $c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-parity > gpurun_out/push${N}.json 2> gpurun_out/push${N}.err
python -c "import json; d=json.load(open('gpurun_out/push${N}.json')); print('[$c]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['launches_per_iteration'], d['collectives'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/push${N}.err
done
