export CFG=${CFG:-2} REPS=2
timeout 600 python tools/prof_scan.py > gpurun_out/plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_scan.py > /dev/null 2>&1; echo rc=$?
