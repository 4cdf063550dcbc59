# scan phase with one vs two query tiles per unit (LV_Q2), flags 0 (normal) and 1 (no top-R work)
for c in ${CFGS:-2 3}; do
  for q in 0 1; do
    echo "== cfg $c q2 $q"
    LV_Q2=$q CFG=$c REPS=5 FLAGS=${FL:-0,1} timeout 300 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
