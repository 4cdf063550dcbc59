# appender probes: clock attribution; entries dropped (256); no list stores (512)
for c in 2 3; do
  LV_LIB=paper_2410_22347_b200/variants/liblv_clk.so CFG=$c REPS=1 FLAGS=128 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
  CFG=$c REPS=3 FLAGS=0,256,512,4 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('cfg', d['cfg'], 'flags', d['flags'], 'main', round(d['main_ms'],4)) for d in map(json.loads, sys.stdin)]"
done
