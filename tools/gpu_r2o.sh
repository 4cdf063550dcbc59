set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_i8.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_r2o.log 2>&1; tail -2 gpurun_out/pytest_r2o.log
LV_LIB=paper_2410_22347_b200/variants/liblv_split.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_i8.py -q -x > gpurun_out/pytest_r2o_split.log 2>&1; tail -2 gpurun_out/pytest_r2o_split.log
VARIANTS="base split" CFGS="2 3 5" REPS=5 bash tools/gpu_variants.sh
LOW=i8 VARIANTS="base split" CFGS="2" REPS=5 bash tools/gpu_variants.sh
