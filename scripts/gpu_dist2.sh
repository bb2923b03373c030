# multi-GPU checks (gpurun --gpus N): dist parity tests, bench at N with the parity leg
N=${1:-2}
mkdir -p gpurun_out
timeout 2700 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/dist${N}_tests.log 2>&1; echo dist_tests_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/dist${N}_tests.log | tail -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/dist${N}_bench.json 2> gpurun_out/dist${N}_bench.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/dist${N}_bench.json')); print(round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['halo_path'], d['launches_per_iteration'], d['parity'], d['roofline']['avg_launch_us'], d['clocks'])"
tail -3 gpurun_out/dist${N}_bench.err
