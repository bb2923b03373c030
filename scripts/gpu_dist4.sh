# 4-GPU evidence (gpurun --gpus 4): dist tests, weak-scaling bench lines at 2 and 4 GPUs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/dist4_tests.log 2>&1; echo dist_tests_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/dist4_tests.log | tail -5
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r02_bench_${N}gpu.json 2> gpurun_out/r02_bench_${N}gpu.err; echo bench_${N}_rc=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_${N}gpu.json')); print(${N}, round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['halo_path'], d['launches_per_iteration'], d['parity']['ok'], d['roofline']['avg_launch_us'], d['clocks'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 5 --warmup 3 --vbm > gpurun_out/r02_bench_4gpu_vbm.json 2> gpurun_out/r02_bench_4gpu_vbm.err; echo vbm4_rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 3 --warmup 2 --global-grid 512 > gpurun_out/r02_bench_4gpu_strong512.json 2> gpurun_out/r02_bench_4gpu_strong512.err; echo strong_rc=$?
python -c "import json; d=json.load(open('gpurun_out/r02_bench_4gpu_strong512.json')); print('strong', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'])"
# replicated-suffix threshold A/B: level 2 (65,000 rows per GPU) replicated too
for N in 2 4; do
PSC_REPL_ROWS=300000 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-kernel-table --no-parity > gpurun_out/r02_bench_${N}gpu_repl300k.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/r02_bench_${N}gpu_repl300k.json')); print('repl300k', ${N}, round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['launches_per_iteration'])"
done
