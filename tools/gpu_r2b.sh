set -x
timeout 900 python -m pytest tests/test_gpu_flex.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_gpu_r2b.log 2>&1
tail -30 gpurun_out/pytest_gpu_r2b.log
for hb in 1 2 1 2; do
LV_HOST_BATCHES=$hb timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_hb$hb.json 2> gpurun_out/bench_hb$hb.err
python -c "import json; d=json.load(open('gpurun_out/bench_hb$hb.json')); print('hb=$hb', d['value'], d['e2e']['value'])"
done
