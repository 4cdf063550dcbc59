# K6 K-block size: 32-element stages (default build) against the 64-element variant (k6kb64), same box;
# the kb64 variant needs its own B-plane tensor maps, so the whole library variant is loaded
OUT=gpurun_out/${OUTDIR:-k6kb}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "g1_encode or mma_exact or full_copy" > $OUT/pytest_g1.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_g1.txt
run() { name=$1; shift; timeout 300 python tools/prof_encode.py --reps 4 "$@" > $OUT/enc_$name.log 2>&1; echo "$name: $(tail -1 $OUT/enc_$name.log)"; }
for v in main k6kb64; do
  if [ $v = main ]; then unset LV_LIB; else export LV_LIB=paper_2410_22347_b200/variants/liblv_$v.so; fi
  run cfg2_$v --n 1000000 --D 512 --d 128 --C 1
  run cfg3_$v --n 1000000 --D 512 --d 96 --C 16
  run cfg4_$v --n 4000000 --D 200 --d 64 --C 1 --low fp16
  run cfg5_$v --n 4000000 --D 768 --d 160 --C 32 --xf16
  LV_K6_HPLANES=3 run cfg5h3_$v --n 4000000 --D 768 --d 160 --C 32 --xf16
done
unset LV_LIB
timeout 600 python tools/k6_flips.py > $OUT/flips_main.txt 2>&1; tail -5 $OUT/flips_main.txt
