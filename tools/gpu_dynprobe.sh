# scan phase with static (LV_DYN_UNITS=0) vs dynamic (1) work-unit order
for c in ${CFGS:-2 3}; do
  for dy in 0 1 0 1; do
    echo "== cfg $c dyn $dy"
    LV_DYN_UNITS=$dy CFG=$c REPS=5 FLAGS=0 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
