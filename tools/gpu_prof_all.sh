# per config: plain run, launch list, one full ncu capture of one lv_search (tools/gpu_prof_full.sh),
# summarised on the box into gpurun_out/prof/ (the .ncu-rep files are deleted: gpurun only brings
# back 64 MiB); then the bench lines (tools/gpu_sweep.sh)
mkdir -p gpurun_out/prof
for c in ${CFGS:-2 3 5}; do
  CFG=$c bash tools/gpu_prof_full.sh
  python tools/ncu_summarize.py --cfg $c --rep gpurun_out/prof_full_cfg$c.ncu-rep --launches gpurun_out/launches_cfg$c.csv \
      --tag ${TAG:-r01} --out gpurun_out/prof > gpurun_out/prof/summ_cfg$c.log 2>&1
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_full_cfg$c.ncu-rep
done
[ -n "$NO_SWEEP" ] || bash tools/gpu_sweep.sh
