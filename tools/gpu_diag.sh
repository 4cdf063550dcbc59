for c in 2 5; do CFG=$c REPS=2 FLAGS=2 timeout 900 python tools/prof_scan.py 2>&1 | grep "sampled"; CFG=$c REPS=2 timeout 900 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\]"; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
