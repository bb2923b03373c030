# A/B of env variants at N GPUs (under gpurun --gpus N), plus the 1-GPU bench on GPU 0
N=${1:-2}; shift
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/dab1.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/dab1.json')); print('[1 GPU]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0])"
i=0
for cfg in "" "$@"; do
i=$((i+1))
env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e > gpurun_out/dab${i}.json 2> gpurun_out/dab${i}.err || { echo "FAIL [$cfg]"; tail -5 gpurun_out/dab${i}.err; continue; }
python -c "import json; d=json.load(open('gpurun_out/dab${i}.json')); print('[$cfg]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], d['halo_path'], d['launches_per_iteration'])"
done
