# round-2 closing run: stride-32 default on the 10M-row configs (full-size parity + bench lines),
# the LV_CHECKS build over the sanitizer cases and parity suites (now with K6 asserts), K6 ncu capture
OUT=gpurun_out/${OUTDIR:-r02f}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "4 or 5" --durations=6 > $OUT/pytest_fullsize_45.txt 2>&1; echo "fullsize rc=$?"; tail -3 $OUT/pytest_fullsize_45.txt
for spec in "5" "4 --family ood" "4 --family id"; do
  name=$(echo "$spec" | tr -d ' -' )
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > $OUT/bench_cfg$name.json 2> $OUT/bench_cfg$name.err
  echo "cfg $spec rc=$?"
  python -c "import json,sys; d=json.load(open('$OUT/bench_cfg$name.json')); k=d['kernel_ms']; print(d['config']['workload'], d['value'], 'e2e', d['e2e']['value'], k, 'frac', d['roofline']['frac'], 'phase', d['scan_phase'].get('frac_of_tensor_peak'), 'recall', d.get('recall_at_10'), d['clocks'])" 2>&1 | tail -1
done
bash tools/gpu_checks.sh > $OUT/checks.log 2>&1; tail -4 $OUT/checks.log; cp gpurun_out/checks_cases.log gpurun_out/checks_pytest.log $OUT/ 2>/dev/null
OUTDIR=${OUTDIR:-r02f}/k6ncu bash tools/gpu_k6_ncu.sh
