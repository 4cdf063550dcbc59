export CFG=2 REPS=1
timeout 600 python tools/prof_scan.py > gpurun_out/plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_score_topr -s 1 -c 1 -o gpurun_out/prof_main python tools/prof_scan.py > gpurun_out/ncu_full.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_full.log
