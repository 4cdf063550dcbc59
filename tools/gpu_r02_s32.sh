# the stride-32 parity test, then stride 16 / 24 / 32 at the 1M-row configs (cheaper appends since the
# split epilogue: does the half-size sample pay there too?)
mkdir -p gpurun_out/s32
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sampled_path" > gpurun_out/s32/pytest_sampled.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s32/pytest_sampled.txt
CFGS=2 SZ="16:2.9 32:2.9 24:2.9 16:2.9 32:2.9" TL=1 FL=0 bash tools/gpu_zsweep.sh
CFGS=3 SZ="16:2.5 32:2.5 24:2.5 16:2.5 32:2.5" TL=1 FL=0 bash tools/gpu_zsweep.sh
