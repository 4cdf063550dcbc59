# one full ncu capture (with source-level warp-state sampling) of the cfg 2 main scan
CFG=2 REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_score_topr" --launch-skip 1 -c 1 -o gpurun_out/app_cfg2 python tools/prof_scan.py > gpurun_out/app_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/app_ncu.log
