# MMA-pipeline probes: scan phase (ms) with no top-R work (flag 1) vs ring depth (LV_STAGES), and
# with accumulators released unread (flag 16, experiment build with -DLV_PROBE_NOLD)
for c in ${CFGS:-2 3}; do
  for st in ${STAGES:-2 3 4 8}; do
    echo "== cfg $c stages $st flags 1"
    LV_STAGES=$st CFG=$c REPS=3 FLAGS=1 timeout 300 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
  echo "== cfg $c nold flags 17"
  LV_LIB=paper_2410_22347_b200/variants/liblv_nold.so CFG=$c REPS=3 FLAGS=1,17 timeout 300 python tools/prof_scan.py 2>/dev/null | grep '^{'
done
