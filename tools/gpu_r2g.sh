set -x
VARIANTS="base dual" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
LOW=i8 VARIANTS="base dual" CFGS="2 5" REPS=5 bash tools/gpu_variants.sh
