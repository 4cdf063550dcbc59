# ncu evidence for one config (CFG, optional LOW=i8): plain run, launch list of one lv_search, one
# full capture of every kernel of one lv_search (+ K6 encode), all on the product path; the reports
# are summarised on the box (gpurun_out/prof/, tag TAGR, default r02) and deleted (gpurun copies
# back at most 64 MiB)
CFG=${CFG:-5}
TAG=cfg$CFG${LOW:+_$LOW}
TAGR=${TAGR:-r02}
export CFG LOW REPS=2
mkdir -p gpurun_out/prof
timeout 900 python tools/prof_scan.py > gpurun_out/prof/plain_$TAG.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$TAG.csv python tools/prof_scan.py > gpurun_out/prof/ncu_list_$TAG.log 2>&1 &&
REPS=1 timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"k_encode_tc|k_proj_tc|k_i8_queries|k_score_topr|k_bmax_select|k_select_topr|k_rerank_topk" -c 14 -o /tmp/prof_$TAG python tools/prof_scan.py > gpurun_out/prof/ncu_full_$TAG.log 2>&1
echo "prof $TAG rc=$?"
python tools/ncu_summarize.py --cfg $CFG ${LOW:+--key cfg${CFG}_$LOW} --rep /tmp/prof_$TAG.ncu-rep --launches gpurun_out/prof/launches_$TAG.csv --tag $TAGR --out gpurun_out/prof > /dev/null 2>&1
echo "summary rc=$?"
rm -f /tmp/prof_$TAG.ncu-rep
tail -2 gpurun_out/prof/plain_$TAG.log
