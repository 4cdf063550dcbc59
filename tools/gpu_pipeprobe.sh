# MMA-pipeline probe: scan phase (ms) with no top-R work (flag 1) vs ring depth (LV_STAGES).
# (The unread-accumulator probe, flag 16, needed a one-off experiment build.)
for c in ${CFGS:-2 3}; do
  for st in ${STAGES:-2 3 4 8}; do
    echo "== cfg $c stages $st flags 1"
    LV_STAGES=$st CFG=$c REPS=3 FLAGS=1 timeout 300 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
