# Variable V-cycle (P:330 footnote) on 1 GPU: parity tests + a bench line at 256^3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variable_v.py -q -x > gpurun_out/varv_tests.log 2>&1; echo varv_tests_rc=$?
tail -2 gpurun_out/varv_tests.log
timeout 900 python bench.py --variable-v --no-cpu-baseline > gpurun_out/varv_bench.json 2> gpurun_out/varv_bench.err; echo varv_bench_rc=$?
tail -c 600 gpurun_out/varv_bench.json
timeout 900 python bench.py --variable-v --vbm --no-cpu-baseline > gpurun_out/varv_vbm_bench.json 2> gpurun_out/varv_vbm_bench.err; echo varv_vbm_bench_rc=$?
tail -c 300 gpurun_out/varv_vbm_bench.json
timeout 900 python bench.py --variable-v --unsmoothed-p --no-cpu-baseline > gpurun_out/varv_tentp_bench.json 2> gpurun_out/varv_tentp_bench.err; echo varv_tentp_bench_rc=$?
tail -c 300 gpurun_out/varv_tentp_bench.json
