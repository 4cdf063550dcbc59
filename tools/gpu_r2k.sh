set -x
./tools/ubench/mma_vs_drain
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check no --report-api-errors no python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"
tail -15 gpurun_out/sanitize_memcheck.log
