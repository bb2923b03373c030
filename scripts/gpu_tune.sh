# layout tuning sweep (under gpurun): prints value per env setting
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for cfg in "" "PSC_RG_DIV=2" "PSC_RG_DIV=8" "PSC_RG_DIV=16" "PSC_RG_MIN=40"; do
  env $cfg $B > gpurun_out/tune.json 2>gpurun_out/tune.err || { echo "FAIL $cfg"; tail -3 gpurun_out/tune.err; continue; }
  python -c "import json,sys; d=json.load(open('gpurun_out/tune.json')); print('$cfg', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], round(d['roofline']['frac'],3))"
done
