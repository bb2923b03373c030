# BASELINE configs at full size on 1 GPU: C2 128^3 (full V-cycle), C5-per-GPU jump 256^3
python bench.py --grid 128 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c2.json 2> gpurun_out/cfg_c2.err; echo c2_rc=$?
python bench.py --problem jump --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/cfg_c5_1gpu.json 2> gpurun_out/cfg_c5_1gpu.err; echo c5_rc=$?
tail -3 gpurun_out/cfg_c5_1gpu.err
for f in cfg_c2 cfg_c5_1gpu; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['config']['levels'], d['config']['rows_rank0'])"; done
