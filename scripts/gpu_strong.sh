# BASELINE configs[3]: 512^3 global, strong scaling over N GPUs (under gpurun --gpus N)
N=${1:-4}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --global-grid 512 --steps 3 --warmup 2 --no-e2e > gpurun_out/strong${N}.json 2> gpurun_out/strong${N}.err; echo "strong rc=$?"
tail -3 gpurun_out/strong${N}.err
python -c "import json; d=json.load(open('gpurun_out/strong${N}.json')); print('[strong $N]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['config']['setup_s'], d['halo_path'])"
