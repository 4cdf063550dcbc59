for c in 3 2; do for f in 4 8 0; do echo "cfg $c flags $f"; CFG=$c REPS=3 FLAGS=$f timeout 900 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"; done; done
