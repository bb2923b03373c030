# same-box A/B of run-time switches on the 1-GPU bench (kernel table per run).
# Usage: gpu_ab.sh TAG "ENV_A" "ENV_B" [reps]
TAG=$1; A=$2; B=$3; REPS=${4:-2}
mkdir -p gpurun_out
for k in $(seq 1 $REPS); do for v in "$A" "$B"; do
  n=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/${TAG}_${n}_$k.json 2> gpurun_out/${TAG}_${n}_$k.err
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_${n}_$k.json')); print('[$v]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['clocks']['sm_mhz'])
for r in d['kernel_table']['rows']:
    if r['level'] in (0,-1) and 'sell' in r['kernel']: print('  ', r['kernel'], r['level'], r['us_per_call'], r['layout_frac'])"
done; done
