set -x
timeout 900 python -m pytest tests/test_gpu_flex.py tests/test_gpu_edges.py -q > gpurun_out/pytest_gpu_r2c.log 2>&1
tail -40 gpurun_out/pytest_gpu_r2c.log
for f in 0 1 33 65 97; do
LV_DEBUG_SCAN_FLAGS=$f timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/probe_c3_f$f.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/probe_c3_f$f.json')); k=d['kernel_ms']; print('flags=$f', 'main', k['main_scan'], 'sample', k['sample_stage'])"
done
for f in 0 1 33 65 97; do
LV_DEBUG_SCAN_FLAGS=$f timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/probe_c2_f$f.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/probe_c2_f$f.json')); k=d['kernel_ms']; print('c2 flags=$f', 'main', k['main_scan'], 'sample', k['sample_stage'])"
done
