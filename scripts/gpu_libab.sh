# A/B of library builds (under gpurun): bash scripts/gpu_libab.sh lib1.so lib2.so ...
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
for lib in "$@"; do
  PSC_LIB=$PWD/paper_2406_19754_b200/$lib $B > gpurun_out/libab.json 2>gpurun_out/libab.err || { echo "FAIL $lib"; tail -3 gpurun_out/libab.err; continue; }
  python -c "import json; d=json.load(open('gpurun_out/libab.json')); print('[$lib]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0])"
done
done
