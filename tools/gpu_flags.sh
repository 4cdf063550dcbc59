# scan ceiling probe: FLAGS=1 makes the epilogue skip top-R (MMA/TMA/TMEM-load throughput only)
free -g | head -2; nproc
for c in ${CFGS:-2 3}; do CFG=$c REPS=3 FLAGS=0,1 timeout 900 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\] gen"; done
