# verify the current build: full GPU suite, smoke, bench lines for configs 5 / 2 / 3
OUT=gpurun_out/${OUTDIR:-r02v}
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.txt
for spec in ${SPECS:-5 2 3}; do
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > $OUT/bench_cfg$spec.json 2> $OUT/bench_cfg$spec.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('$OUT/bench_cfg$spec.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], 'main', k['main_scan'], 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'K5', d['roofline_rerank']['frac'], 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
