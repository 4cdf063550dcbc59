# round-2 evidence on the current build: full GPU suite, smoke, bench lines (cfg 5 default, 2, 3),
# launch list + full ncu capture per config
mkdir -p gpurun_out/r02f
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02f/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02f/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02f/smoke.txt
for spec in "5" "2" "3"; do
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > gpurun_out/r02f/bench_cfg$spec.json 2> gpurun_out/r02f/bench_cfg$spec.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r02f/bench_cfg$spec.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], 'main', k['main_scan'], 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'K5', d['roofline_rerank']['frac'], 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
for c in 2 3 5; do CFG=$c bash tools/gpu_prof_r02.sh; done
