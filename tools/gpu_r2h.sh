set -x
timeout 600 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -12 gpurun_out/sanitize_plain.log
VARIANTS="base tree" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
for low in bf16 i8; do
for f in 2 4; do
echo "== cfg2 $low flags $f"
LOW=$low CFG=2 REPS=2 FLAGS=$f timeout 600 python tools/prof_scan.py 2>&1 | grep "^\[lv\] main\|^{" | tail -3
done
done
