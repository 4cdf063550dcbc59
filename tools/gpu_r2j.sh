set -x
VARIANTS="base epispin mmaspin bothspin" CFGS="2 3" REPS=5 FL=0,1 bash tools/gpu_variants.sh
LOW=i8 VARIANTS="base" CFGS="2" REPS=5 bash tools/gpu_variants.sh
