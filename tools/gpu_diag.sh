timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for f in 1 4 0; do CFG=2 REPS=3 FLAGS=$f timeout 600 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"; done
CFG=3 REPS=3 timeout 600 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"
