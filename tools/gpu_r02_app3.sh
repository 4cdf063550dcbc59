# appender with mbarrier ring handshake: quick parity, scan timings, counts, clock attribution
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_i8.py -x -q 2>&1 | tail -2
VARIANTS="base" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
for c in 2 3; do
  CFG=$c REPS=1 FLAGS=2 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
  LV_LIB=paper_2410_22347_b200/variants/liblv_clk.so CFG=$c REPS=1 FLAGS=128 timeout 600 python tools/prof_scan.py 2>&1 | grep -E "^\[lv\] main"
done
