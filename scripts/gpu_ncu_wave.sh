#!/bin/bash
mkdir -p gpurun_out
T=${1:-ncuwave}
PSC_WAVE=1 timeout 600 python bench.py --steps 1 --warmup 0 --grid 128 --no-cpu-baseline --no-e2e > gpurun_out/${T}_plain.json 2>&1; echo "plain_rc=$?"
PSC_WAVE=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^sell_wave$ -s 1 -c 1 -o gpurun_out/${T} python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sell_tma -s 12 -c 1 -o gpurun_out/${T}_tma python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu2.log 2>&1; echo "ncu2_rc=$?"
