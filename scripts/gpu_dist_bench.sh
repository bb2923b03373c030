N=${1:-2}; CFG=$2
env $CFG timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e > gpurun_out/db_${N}.json 2> gpurun_out/db_${N}.err; echo "bench [$CFG] rc=$?"
grep -v OMP gpurun_out/db_${N}.err | tail -40
cat gpurun_out/db_${N}.json
