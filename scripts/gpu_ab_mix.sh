B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
for cfg in "" "PSC_NO_DINV_FLY=1" "PSC_LIB=$PWD/paper_2406_19754_b200/libpsc_noex.so"; do
  env $cfg $B > gpurun_out/mix.json 2>gpurun_out/mix.err || { echo "FAIL $cfg"; tail -3 gpurun_out/mix.err; continue; }
  python -c "import json; d=json.load(open('gpurun_out/mix.json')); print('[${cfg##*/}]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], round(d['roofline']['avg_launch_us'],1))"
done; done
