# K6 encode: G1 parity of every encode shape + the X_full copy, then timing at the cfg 2 / 3 / 4 / 5
# shapes; fp16 rows: direct with 2 / 3 planes (LV_K6_HPLANES) or as three bf16 planes (LV_K6_DIRECT=0)
OUT=gpurun_out/${OUTDIR:-k6}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "g1_encode or mma_exact or full_copy" > $OUT/pytest_g1.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_g1.txt
run() { name=$1; shift; timeout 300 python tools/prof_encode.py "$@" > $OUT/enc_$name.log 2>&1; echo "$name: $(tail -1 $OUT/enc_$name.log)"; }
C5="--n 4000000 --D 768 --d 160 --C 32 --xf16"
run cfg2 --n 1000000 --D 512 --d 128 --C 1
run cfg3 --n 1000000 --D 512 --d 96 --C 16
run cfg4 --n 4000000 --D 200 --d 64 --C 1 --low fp16
run cfg5 $C5
LV_K6_HPLANES=3 run cfg5_h3 $C5
LV_K6_DIRECT=0 run cfg5_bf16planes $C5
