set -x
timeout 900 python -m pytest tests/test_gpu_i8.py -q -x > gpurun_out/pytest_gpu_r2e.log 2>&1
tail -40 gpurun_out/pytest_gpu_r2e.log
timeout 600 python bench.py --config 2 --low i8 --steps 10 --warmup 3 --oracle-queries 50 > gpurun_out/bench_c2_i8.json 2> gpurun_out/bench_c2_i8.err; tail -3 gpurun_out/bench_c2_i8.err
python -c "import json; d=json.load(open('gpurun_out/bench_c2_i8.json')); print(d['value'], d['kernel_ms'], d['roofline']['frac'], d['recall_at_10'])"
