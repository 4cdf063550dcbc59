# scan phase vs the number of database chunks (units = chunks x query tiles; fewer, longer units)
for c in ${CFGS:-2 3}; do
  for mc in ${MCS:-1000000000 60 30}; do
    echo "== cfg $c max_chunks $mc"
    LV_MAX_CHUNKS=$mc CFG=$c REPS=5 FLAGS=0 timeout 300 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
