# (record of a round-2 experiment: the LV_K6_NOFULL / LV_K6_NOPF code paths it selected were removed after the measurement)
# K6 A/B on one box: default build with the fused copy / L2 prefetch toggled by environment, and the
# variant builds k6base (neither compiled in) and k6ring3 (fp32 register ring of 3 blocks, no fused copy)
OUT=gpurun_out/${OUTDIR:-k6ab}
mkdir -p $OUT
run() { name=$1; shift; timeout 300 python tools/prof_encode.py --reps 4 "$@" > $OUT/enc_$name.log 2>&1; echo "$name: $(tail -1 $OUT/enc_$name.log)"; }
C2="--n 1000000 --D 512 --d 128 --C 1"
C4="--n 4000000 --D 200 --d 64 --C 1 --low fp16"
C5="--n 4000000 --D 768 --d 160 --C 32 --xf16"
V=paper_2410_22347_b200/variants
for rep in 1 2; do
for c in 2 4 5; do
  eval "S=\$C$c"
  LV_LIB=$V/liblv_k6base.so LV_K6_FUSE_COPY=0 run cfg${c}_base_$rep $S
  LV_K6_FUSE_COPY=0 LV_K6_L2PF=0 run cfg${c}_nofuse_nopf_$rep $S
  LV_K6_FUSE_COPY=0 run cfg${c}_nofuse_pf_$rep $S
  LV_K6_L2PF=0 run cfg${c}_fuse_nopf_$rep $S
  run cfg${c}_fuse_pf_$rep $S
  LV_LIB=$V/liblv_k6ring3.so LV_K6_FUSE_COPY=0 LV_K6_L2PF=0 run cfg${c}_ring3_nopf_$rep $S
  LV_LIB=$V/liblv_k6ring3.so LV_K6_FUSE_COPY=0 run cfg${c}_ring3_pf_$rep $S
done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
