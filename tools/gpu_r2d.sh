set -x
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q --durations=10 > gpurun_out/pytest_fullsize_r2d.log 2>&1
tail -30 gpurun_out/pytest_fullsize_r2d.log
