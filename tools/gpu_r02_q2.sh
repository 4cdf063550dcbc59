# quick check of the pending changes: parity subset, scan timings, counts, bench e2e with host batches 2 / 4 / 8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_i8.py tests/test_gpu_flex.py -x -q 2>&1 | grep -E "FAILED|Error|passed|failed" | head -20
for c in 2 3; do
  CFG=$c REPS=5 FLAGS=0 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('cfg', d['cfg'], 'flags', d['flags'], 'main', round(d['main_ms'],4), {k: round(v,3) for k,v in d['kernel_ms'].items()}) for d in map(json.loads, sys.stdin)]"
  CFG=$c REPS=1 FLAGS=2 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
done
for hb in 2; do break
  LV_HOST_BATCHES=$hb timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --oracle-queries 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('hb $hb', d['value'], 'e2e', d['e2e']['value'], d['clocks']['sm_mhz'])"
done
