# Memory-safety evidence without compute-sanitizer (closed on this pool): the LV_CHECKS build (device
# bounds asserts in the scan, K4 and K5; every source rebuilt with -DLV_CHECKS) runs the sanitizer
# cases and the GPU parity suites; any failed check traps the kernel and fails the run.
set -x
test -f paper_2410_22347_b200/variants/liblv_checks.so || exit 1   # built here: VARIANT_SRC=all python tools/build_variant.py checks -DLV_CHECKS
export LV_LIB=paper_2410_22347_b200/variants/liblv_checks.so
timeout 900 python tools/sanitize_cases.py > gpurun_out/checks_cases.log 2>&1; echo "cases rc=$?"; tail -12 gpurun_out/checks_cases.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_i8.py tests/test_gpu_flex.py -q > gpurun_out/checks_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/checks_pytest.log
grep -c "LV_CHECK failed" gpurun_out/checks_cases.log gpurun_out/checks_pytest.log
