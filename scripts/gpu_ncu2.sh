# two full ncu captures (under gpurun): level-0 sweep (sell_tma<Sweep>) and level-1 sweep (rg_tma<Sweep,4>)
TAG=${1:-n}
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$SMALL > gpurun_out/${TAG}_plain.log 2>&1 || { echo plain failed; exit 1; }
true
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:rg_tma<\(psc::RowOp\)2, \(int\)4>' -c 2 -o gpurun_out/${TAG}_l1 $SMALL > gpurun_out/${TAG}_l1.log 2>&1; echo l1_rc=$?
tail -3 gpurun_out/${TAG}_l0.log gpurun_out/${TAG}_l1.log
