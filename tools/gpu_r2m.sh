set -x
LV_LIB=paper_2410_22347_b200/variants/liblv_hitlocal.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_i8.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_r2m.log 2>&1; tail -3 gpurun_out/pytest_r2m.log
VARIANTS="base hitlocal" CFGS="2 3 5" REPS=5 bash tools/gpu_variants.sh
LOW=i8 VARIANTS="base hitlocal" CFGS="2" REPS=5 bash tools/gpu_variants.sh
for c in 2 3; do
LV_LIB=paper_2410_22347_b200/variants/liblv_hitlocalclk.so LV_DEBUG_SCAN_FLAGS=128 CFG=$c REPS=1 FLAGS=128 timeout 600 python tools/prof_scan.py 2>&1 | grep "^\[lv\] main"
done
