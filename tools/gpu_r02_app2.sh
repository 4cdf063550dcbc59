# appender attribution: base vs sleeping epilogue waits, event counts (flag 2), clock probe (flag 128)
VARIANTS="base sleep" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
for c in 2 3; do
  CFG=$c REPS=1 FLAGS=2 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] (main|sample)"
  LV_LIB=paper_2410_22347_b200/variants/liblv_clk.so CFG=$c REPS=1 FLAGS=128 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
done
