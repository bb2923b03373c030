# same-box A/B of run-time switches on the N-GPU bench.  Usage: gpu_ab_dist.sh N TAG "ENV_A" "ENV_B" [reps]
N=$1; TAG=$2; A=$3; B=$4; REPS=${5:-1}
mkdir -p gpurun_out
for k in $(seq 1 $REPS); do for v in "$A" "$B"; do
  n=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 5 --warmup 3 --no-parity --no-e2e \
    > gpurun_out/${TAG}_${n}_$k.json 2> gpurun_out/${TAG}_${n}_$k.err
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_${n}_$k.json')); print('[$v]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in (d.get('kernel_table') or {}).get('rows', []):
    if r['level'] in (0,-1) and 'sell' in r['kernel']: print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'])" || tail -3 gpurun_out/${TAG}_${n}_$k.err
done; done
