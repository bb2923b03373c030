# multi-GPU checks (under gpurun --gpus N): dist parity tests + bench at N
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist${N}_tests.log 2>&1; echo dist_tests_rc=$?
tail -30 gpurun_out/dist${N}_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 3 --warmup 2 --no-e2e > gpurun_out/dist${N}_bench.json 2> gpurun_out/dist${N}_bench.err; echo bench_rc=$?
tail -5 gpurun_out/dist${N}_bench.err; cat gpurun_out/dist${N}_bench.json
