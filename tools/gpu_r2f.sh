set -x
./tools/ubench/tmem_drain
timeout 900 python -m pytest tests/test_gpu_i8.py -q > gpurun_out/pytest_gpu_r2f.log 2>&1
tail -30 gpurun_out/pytest_gpu_r2f.log
for f in 1 65; do
LV_DEBUG_SCAN_FLAGS=$f timeout 600 python bench.py --config 2 --low i8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/probe_c2i8_f$f.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/probe_c2i8_f$f.json')); k=d['kernel_ms']; print('c2 i8 flags=$f', 'main', k['main_scan'], 'sample', k['sample_stage'])"
done
