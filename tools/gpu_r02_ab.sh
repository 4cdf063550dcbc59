# A/B: accumulator wait by spinning (base) vs suspend-hint sleep (LV_EPI_SLEEP)
VARIANTS="base sleep" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
VARIANTS="sleep base" CFGS="2 3" REPS=5 bash tools/gpu_variants.sh
