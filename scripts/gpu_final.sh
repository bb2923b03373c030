# Round evidence (under gpurun, 1 GPU): smoke, every GPU test, the bench line, the
# reference arm, and the other configurations' lines.  TAG = round tag.
TAG=${1:-r02f}
mkdir -p gpurun_out
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo tests_rc=$?
tail -2 gpurun_out/${TAG}_gpu_tests.log
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt
PSC_AMG_VERBOSE=1 timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?; grep psc_amg gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref_rc=$?
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-kernel-table"
for cfg in "--vbm" "--vbm --hierarchy smatch" "--vbm --hierarchy vmatch" "--variable-v" "--problem jump" "--grid 128" "--setup host" "--smoother ainv"; do
  name=$(echo "$cfg" | tr -d ' -' )
  timeout 900 $B $cfg > gpurun_out/${TAG}_bench_${name}.json 2> gpurun_out/${TAG}_bench_${name}.err; echo "$cfg rc=$?"
done
for f in gpurun_out/${TAG}_bench*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d.get('metric'), round(d.get('value',0),1), d.get('ms_per_step'), (d.get('config') or {}).get('iters',[None])[0], (d.get('clocks') or {}).get('sm_mhz'))" 2>/dev/null; done
