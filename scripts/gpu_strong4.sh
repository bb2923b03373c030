# strong-scaling check on 4 GPUs (+ the halo-poison parity variants)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "POISON" > gpurun_out/strong4_tests.log 2>&1; echo poison_rc=$?; tail -2 gpurun_out/strong4_tests.log
for G in 256 512; do
PSC_SPIN_TIMEOUT_S=240 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 3 --warmup 2 --global-grid $G --no-kernel-table > gpurun_out/strong4_${G}.json 2> gpurun_out/strong4_${G}.err; echo strong_${G}_rc=$?
python -c "import json; d=json.load(open('gpurun_out/strong4_${G}.json')); print('strong', ${G}, round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['config']['setup_s'])" 2>/dev/null || grep -E "PscError|Error" gpurun_out/strong4_${G}.err | head -4
done
