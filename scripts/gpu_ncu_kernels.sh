# ncu evidence for the per-kernel table (1 GPU): launch list of one solve, then one
# --set full capture of every distinct kernel of the first iteration (256^3 bench config)
TAG=${1:-r02}
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kernel-table"
$SMALL > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err; echo plain_rc=$?
PSC_PROFILE_SOLVE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
# one full capture per kernel family of the first iteration (ordered launches 0..~40)
PSC_PROFILE_SOLVE=1 timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on -c 40 -o /tmp/${TAG}_kernels $SMALL > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full_rc=$?
python scripts/ncu_summary.py /tmp/${TAG}_kernels.ncu-rep > gpurun_out/${TAG}_ncu_kernels.txt 2>&1; echo sum_rc=$?
python scripts/summarize_launches.py gpurun_out/${TAG}_launches.csv --by-grid > gpurun_out/${TAG}_launches.txt 2>&1
head -30 gpurun_out/${TAG}_launches.txt
