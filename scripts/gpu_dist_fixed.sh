# per-iteration cost at fixed iteration count (tol 0, maxit K): 1 GPU vs N GPUs, with/without halo traffic
N=${1:-2}; K=${2:-20}
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --tol 0 --maxit $K > gpurun_out/dfx1.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/dfx1.json')); print('[1 GPU]', round(d['ms_per_step']/$K,3), 'ms/it')"
i=0
for cfg in "" "PSC_REPL_ROWS=0" "PSC_NO_P2P=1" "PSC_DEBUG_SKIP_HALO=1"; do
i=$((i+1))
env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e --tol 0 --maxit $K > gpurun_out/dfx${i}.json 2> gpurun_out/dfx${i}.err || { echo "FAIL [$cfg]"; tail -5 gpurun_out/dfx${i}.err; continue; }
python -c "import json; d=json.load(open('gpurun_out/dfx${i}.json')); print('[$cfg]', round(d['ms_per_step']/$K,3), 'ms/it', d['halo_path'], d['launches_per_iteration'])"
done
