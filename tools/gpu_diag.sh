timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 3; do CFG=$c REPS=3 timeout 600 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"; done
