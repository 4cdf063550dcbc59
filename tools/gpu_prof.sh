# ncu evidence for one config (default cfg 2): launch list + full capture of the scan and re-rank kernels
CFG=${CFG:-2}
export CFG REPS=3
timeout 600 python tools/prof_scan.py > gpurun_out/plain_cfg$CFG.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv python tools/prof_scan.py > gpurun_out/ncu_list.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_score_topr|k_select_rerank|k_tau_merge|k_rows_gemm" -s 14 -c 11 -o gpurun_out/prof_cfg$CFG python tools/prof_scan.py > gpurun_out/ncu_full.log 2>&1
echo rc=$?
tail -3 gpurun_out/plain_cfg$CFG.log gpurun_out/ncu_full.log
