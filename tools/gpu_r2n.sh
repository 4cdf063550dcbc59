set -x
bash tools/gpu_checks.sh
timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_gpu_all.log 2>&1; echo "all gpu rc=$?"; tail -18 gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2.log 2>&1; tail -2 gpurun_out/smoke_r2.log
