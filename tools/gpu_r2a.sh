set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:randomly --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1
tail -40 gpurun_out/pytest_gpu_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --oracle-queries 50 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -5 gpurun_out/bench_r2a.err; cat gpurun_out/bench_r2a.json
