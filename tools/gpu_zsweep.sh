# sampled-threshold knobs: scan phase time and hit statistics per (cfg, stride, z)
# SZ="16:2.9 8:2.9" (stride:z pairs), FL=flags list, TL=lines kept per run
for c in ${CFGS:-2 3}; do
  for sz in ${SZ:-16:2.9 16:2.0 8:2.9 8:2.0 32:2.9}; do
    st=${sz%%:*}; z=${sz##*:}
    echo "== cfg $c stride $st z $z"
    CFG=$c REPS=3 FLAGS=${FL:-0,2} LV_SAMPLE_STRIDE=$st LV_SAMPLE_Z=$z timeout 300 python tools/prof_scan.py 2>&1 | grep -E '^\{|\[lv\]' | tail -${TL:-5}
  done
done
