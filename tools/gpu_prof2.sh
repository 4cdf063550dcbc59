export CFG=${CFG:-2} REPS=1
timeout 600 python tools/prof_scan.py > gpurun_out/plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_select_rerank -s 0 -c 1 -o gpurun_out/prof_rerank_cfg$CFG python tools/prof_scan.py > gpurun_out/ncu_rr.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_score_topr|k_proj_tc|k_bmax" -s 0 -c 4 -o gpurun_out/prof_scan_cfg$CFG python tools/prof_scan.py > gpurun_out/ncu_sc.log 2>&1
echo rc=$?; tail -1 gpurun_out/ncu_rr.log gpurun_out/ncu_sc.log
