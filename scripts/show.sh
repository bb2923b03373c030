TAG=$1
python -c "
import json
for f in ('${TAG}_bench','${TAG}_bench_nodia'):
  try:
    d=json.load(open(f'gpurun_out/{f}.json')); print(f, round(d['value'],1), round(d['ms_per_step'],2), d['config']['iters'][0], round(d['roofline']['achieved'] or 0), round(d['roofline']['avg_launch_us'] or 0,1))
  except Exception as e: print(f, 'ERR', e)"
python scripts/summarize_launches.py gpurun_out/${TAG}_launches.csv 2>/dev/null | head -${2:-16}
