N=${1:-2}
for cfg in "PSC_DEBUG_EX=0" "PSC_DEBUG_EX=1" "PSC_DEBUG_EX=2" "PSC_DEBUG_EX=4" "PSC_DEBUG_EX=7" "PSC_NO_P2P=1"; do
env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) scripts/exbench_worker.py 2>/dev/null | grep env
done
