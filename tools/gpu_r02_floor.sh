# floors of the current scan: full, hits detected but not pushed (4), MMA + drain only (1), no TMA (32), one K step (64)
for c in 2 3; do
  CFG=$c REPS=5 FLAGS=0,4,1,65 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('cfg', d['cfg'], 'flags', d['flags'], 'main', round(d['main_ms'],4)) for d in map(json.loads, sys.stdin)]"
done
