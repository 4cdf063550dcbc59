# decoupled append warps: GPU parity suites (without the full-size checks), then bench lines for
# configs 2 / 3 and the scan attribution counters
mkdir -p gpurun_out/r02app
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py > gpurun_out/r02app/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02app/pytest_gpu.txt
for spec in "2" "3"; do
  timeout 900 python bench.py --config $spec --steps 20 --warmup 5 > gpurun_out/r02app/bench_cfg$spec.json 2> gpurun_out/r02app/bench_cfg$spec.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r02app/bench_cfg$spec.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], 'main', k['main_scan'], 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'K5', d['roofline_rerank']['frac'], 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
