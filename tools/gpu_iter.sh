# one build->measure iteration: GPU parity suite, smoke, scan probe (cfg 2/3), short bench
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in ${CFGS:-2 3}; do CFG=$c REPS=3 FLAGS=0,1 timeout 900 python tools/prof_scan.py 2>&1 | grep -v "^\[bench\] gen"; done
timeout 900 python bench.py --steps 10 --warmup 3 --oracle-queries 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
