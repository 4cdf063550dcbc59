# K6: fewer hh accumulators per tile (variant builds k6nh1 / k6nh2) leave TMEM room for a second
# accumulator buffer (d = 128: nH = 1 -> 2 x 2 x 128 columns; d = 96: nH = 1): time and G1 flips
OUT=gpurun_out/${OUTDIR:-k6nh}
mkdir -p $OUT
V=paper_2410_22347_b200/variants
run() { name=$1; shift; timeout 300 python tools/prof_encode.py --reps 4 "$@" > $OUT/enc_$name.log 2>&1; echo "$name: $(tail -1 $OUT/enc_$name.log)"; }
for v in main k6nh1 k6nh2; do
  if [ $v = main ]; then unset LV_LIB; else export LV_LIB=$V/liblv_$v.so; fi
  run cfg2_$v --n 1000000 --D 512 --d 128 --C 1
  run cfg3_$v --n 1000000 --D 512 --d 96 --C 16
  run cfg5_$v --n 4000000 --D 768 --d 160 --C 32 --xf16
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "g1_encode" > $OUT/pytest_$v.txt 2>&1; echo "pytest $v rc=$?"; tail -2 $OUT/pytest_$v.txt
  timeout 600 python tools/k6_flips.py > $OUT/flips_$v.txt 2>&1; tail -4 $OUT/flips_$v.txt
done
