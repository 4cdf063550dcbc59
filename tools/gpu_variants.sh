# scan phase per experiment build (paper_2410_22347_b200/variants/liblv_<name>.so) and config
for v in ${VARIANTS:-base}; do
  for c in ${CFGS:-2 3}; do
    echo "== $v cfg $c"
    LV_LIB=paper_2410_22347_b200/variants/liblv_$v.so CFG=$c REPS=${REPS:-3} FLAGS=${FL:-0} timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{'
  done
done
