set -x
VARIANTS="base onelam" CFGS="2 3" REPS=7 bash tools/gpu_variants.sh
VARIANTS="onelam base" CFGS="2 3" REPS=7 bash tools/gpu_variants.sh
