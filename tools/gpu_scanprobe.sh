# scan-phase breakdown: flags 0 (normal), 1 (no top-R: MMA + TMEM drain only), 4 (hits detected, dropped)
for c in ${CFGS:-2 3 4}; do
  echo "== cfg $c"
  CFG=$c REPS=3 FLAGS=0,1,4 timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{'
done
