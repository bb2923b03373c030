# exchange microbenchmark variants (gpurun --gpus N)
N=${1:-2}
mkdir -p gpurun_out
run() { env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) scripts/exchange_bench.py 2>>gpurun_out/xb.err | tail -1; }
run PSC_P2P_FENCE=0
run PSC_P2P_FENCE=1
run PSC_P2P_FENCE=0 PSC_P2P_BX=8
run PSC_P2P_FENCE=1 PSC_P2P_BX=8
run PSC_P2P_FENCE=1 PSC_P2P_BX=16 PSC_P2P_PER_CTA=1024
run PSC_P2P_FENCE=0 PSC_P2P_BX=1
run PSC_P2P_FENCE=1 PSC_P2P_BX=1
run PSC_P2P_FENCE=0
