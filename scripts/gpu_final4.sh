# Round-end multi-GPU evidence (gpurun --gpus 4): every dist test, weak-scaling lines at
# 2 and 4 GPUs (default, VBM, AINV), strong scaling 512^3 on 4 GPUs.  TAG = round tag.
TAG=${1:-r02f}
mkdir -p gpurun_out
run() {  # N out args...
  local N=$1 o=$2; shift 2
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N "$@" > gpurun_out/${TAG}_$o.json 2> gpurun_out/${TAG}_$o.err
  echo "$o rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/${TAG}_$o.json')); p=d.get('parity') or {}
print('  ', round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'], d['launches_per_iteration'], p.get('ok'), d['roofline']['avg_launch_us'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null
}
[ -z "$SKIP_TESTS" ] && { timeout 2400 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/${TAG}_dist4_tests.log 2>&1; echo dist_tests_rc=$?; }
tail -1 gpurun_out/${TAG}_dist4_tests.log
run 2 bench_2gpu --steps 5 --warmup 3
run 4 bench_4gpu --steps 5 --warmup 3
run 4 bench_4gpu_vbm --steps 5 --warmup 3 --vbm --no-kernel-table
run 4 bench_4gpu_ainv --steps 5 --warmup 3 --smoother ainv --no-kernel-table
run 4 bench_4gpu_strong512 --steps 3 --warmup 3 --global-grid 512 --no-kernel-table
