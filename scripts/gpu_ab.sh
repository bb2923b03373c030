# A/B perf over env variants (under gpurun): bash scripts/gpu_ab.sh TAG "ENV1" "ENV2" ...
TAG=$1; shift
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for cfg in "" "$@"; do
  env $cfg $B > gpurun_out/${TAG}_ab.json 2>gpurun_out/${TAG}_ab.err || { echo "FAIL [$cfg]"; tail -3 gpurun_out/${TAG}_ab.err; continue; }
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_ab.json')); print('[$cfg]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0])"
done
