# round-2 bench lines for every config (plus the int8 lines), one process each
set -x
mkdir -p gpurun_out/r02
for spec in "5" "2" "3" "1" "4 --family ood" "4 --family id" "2 --low i8" "5 --low i8"; do
  name=$(echo "$spec" | tr -d ' -' )
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > gpurun_out/r02/bench_cfg$name.json 2> gpurun_out/r02/bench_cfg$name.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r02/bench_cfg$name.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], 'main', k['main_scan'], 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'K5', d['roofline_rerank']['frac'], 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
