# A/B: shared append rings (base) vs per-warp private rings (priv), interleaved
VARIANTS="base priv" CFGS="2 3" REPS=7 bash tools/gpu_variants.sh
VARIANTS="priv base" CFGS="2 3" REPS=7 bash tools/gpu_variants.sh
