# round-2 baseline on a fresh box: GPU suite (without the full-size checks), smoke, bench lines
# for configs 5 / 2 / 3, launch list + full ncu capture of config 5
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py > gpurun_out/r02/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02/smoke.txt
for spec in "5" "2" "3"; do
  name=$(echo "$spec" | tr -d ' -' )
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > gpurun_out/r02/bench_cfg$name.json 2> gpurun_out/r02/bench_cfg$name.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r02/bench_cfg$name.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], 'main', k['main_scan'], 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'K5', d['roofline_rerank']['frac'], 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
CFG=5 bash tools/gpu_prof_r02.sh
