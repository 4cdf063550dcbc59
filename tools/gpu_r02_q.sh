# quick check: parity subset, scan timings and floors, clock attribution
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_i8.py -x -q 2>&1 | grep -E "FAILED|Error|passed|failed" | head -20
for c in 2 3; do
  CFG=$c REPS=5 FLAGS=${FL:-0,4} timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('cfg', d['cfg'], 'flags', d['flags'], 'main', round(d['main_ms'],4), 'phase', [round(x,3) for x in d['phase_ms']]) for d in map(json.loads, sys.stdin)]"
  LV_LIB=paper_2410_22347_b200/variants/liblv_clk.so CFG=$c REPS=1 FLAGS=128 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
done
