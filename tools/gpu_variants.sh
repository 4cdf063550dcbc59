# scan phase per experiment build (paper_2410_22347_b200/variants/liblv_<name>.so) and config
for v in ${VARIANTS:-base}; do
  for c in ${CFGS:-2 3}; do
    echo "== $v cfg $c"
    lib=paper_2410_22347_b200/variants/liblv_$v.so
    [ "$v" = base ] && lib=paper_2410_22347_b200/liblv.so
    LV_LIB=$lib LOW=${LOW:-} CFG=$c REPS=${REPS:-5} FLAGS=${FL:-0} timeout 600 python tools/prof_scan.py 2>/dev/null | grep '^{' | python -c "import sys,json; [print('$v', 'cfg', d['cfg'], d['low'], 'flags', d['flags'], 'main', round(d['main_ms'],4), 'phase', [round(x,3) for x in d['phase_ms']]) for d in map(json.loads, sys.stdin)]"
  done
done
