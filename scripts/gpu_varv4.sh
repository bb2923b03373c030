# Variable V-cycle on 4 GPUs: distributed parity (4 ranks) + weak-scaling bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -k "four_gpu" > gpurun_out/varv_dist4.log 2>&1; echo dist4_rc=$?; tail -2 gpurun_out/varv_dist4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 4 --steps 5 --warmup 3 --variable-v > gpurun_out/varv_bench4.json 2> gpurun_out/varv_bench4.err; echo bench4_rc=$?
tail -c 400 gpurun_out/varv_bench4.json
