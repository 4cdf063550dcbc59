timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
LV_CPT=64 timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 2 4; do for cpt in 32 64; do echo "cfg $c cpt $cpt"; LV_CPT=$cpt CFG=$c REPS=3 timeout 900 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"; done; done
