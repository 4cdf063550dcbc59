# evidence for one config: plain run, launch list, one full capture of every kernel of one lv_search
export CFG=${CFG:-2} REPS=2
timeout 900 python tools/prof_scan.py > gpurun_out/plain_cfg$CFG.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv python tools/prof_scan.py > /dev/null 2>&1 &&
REPS=1 timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"k_split3|k_encode_tc|k_proj_tc|k_score_topr|k_bmax_select|k_select_topr|k_rerank_topk" -c 12 -o gpurun_out/prof_full_cfg$CFG python tools/prof_scan.py > gpurun_out/ncu_full_cfg$CFG.log 2>&1
echo rc=$?
