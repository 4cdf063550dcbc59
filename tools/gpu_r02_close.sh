# final round-2 evidence on the final build: ncu launch list + full capture at cfg 5 (stride 32),
# then the whole GPU suite, smoke and the default bench line plus configs 2 and 3
CFG=5 bash tools/gpu_prof_r02.sh
OUTDIR=r02final SPECS="5 2 3" bash tools/gpu_r02_verify.sh
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02final/bench_reference_cfg5.json 2> gpurun_out/r02final/bench_reference_cfg5.err; echo "reference rc=$?"; tail -c 600 gpurun_out/r02final/bench_reference_cfg5.json
