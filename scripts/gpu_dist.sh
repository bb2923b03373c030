# multi-GPU checks (under gpurun --gpus N): dist parity tests + bench at N (P2P and NCCL halo paths)
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -30 gpurun_out/dist${N}_tests.log | grep -v "^$" | tail -12
i=0
for cfg in "" "PSC_NO_P2P=1"; do
i=$((i+1))
env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e > gpurun_out/dist${N}_bench${i}.json 2> gpurun_out/dist${N}_bench${i}.err; echo "bench [$cfg] rc=$?"
python -c "import json; d=json.load(open('gpurun_out/dist${N}_bench${i}.json')); print('[$cfg]', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['halo_path'], d['launches_per_iteration'])"
done
