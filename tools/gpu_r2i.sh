set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_i8.py -q -x -k "exact or g1 or shapes or sampled or gleanvec" > gpurun_out/pytest_r2i.log 2>&1; tail -5 gpurun_out/pytest_r2i.log
VARIANTS="base fullacc" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
LOW=i8 VARIANTS="base" CFGS="2" REPS=5 bash tools/gpu_variants.sh
for f in 1 65; do LV_DEBUG_SCAN_FLAGS=$f CFG=2 REPS=3 FLAGS=$f timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('base cfg2 flags', d['flags'], 'main', round(d['main_ms'],4)) for d in map(json.loads, sys.stdin)]"; done
