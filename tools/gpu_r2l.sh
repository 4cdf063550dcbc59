set -x
for c in 2 3; do
for f in 128; do
echo "== cfg $c flags $f"
LV_LIB=paper_2410_22347_b200/variants/liblv_clk.so LV_DEBUG_SCAN_FLAGS=$f CFG=$c REPS=1 FLAGS=$f timeout 600 python tools/prof_scan.py 2>&1 | grep "^\[lv\] main"
done
done
