# scan phase vs the planner's unit-boundary cost (LV_UNIT_COST, in tiles)
for c in ${CFGS:-2 3}; do
  for uc in ${UCS:-2 4 8 16}; do
    echo "== cfg $c unit_cost $uc"
    LV_UNIT_COST=$uc CFG=$c REPS=5 FLAGS=0 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
