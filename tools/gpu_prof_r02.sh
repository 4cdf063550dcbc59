# ncu evidence for one config (CFG, optional LOW=i8): plain run, launch list of one lv_search, one
# full capture of every kernel of one lv_search (+ K6 encode), all on the product path.
CFG=${CFG:-5}
TAG=cfg$CFG${LOW:+_$LOW}
export CFG LOW REPS=2
timeout 900 python tools/prof_scan.py > gpurun_out/plain_$TAG.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_scan.py > gpurun_out/ncu_list_$TAG.log 2>&1 &&
REPS=1 timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"k_encode_tc|k_proj_tc|k_i8_queries|k_score_topr|k_bmax_select|k_select_topr|k_rerank_topk" -c 14 -o gpurun_out/prof_$TAG python tools/prof_scan.py > gpurun_out/ncu_full_$TAG.log 2>&1
echo "prof $TAG rc=$?"
tail -2 gpurun_out/plain_$TAG.log
