# K6 encode: G1 parity of every encode shape, then timing at the cfg 2 / 3 / 5 shapes
# (persistent kernel; fp16 rows: direct fp16 operand against scaled fp16 B planes, A/B LV_K6_DIRECT=0)
OUT=gpurun_out/${OUTDIR:-k6}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "g1_encode or mma_exact" > $OUT/pytest_g1.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_g1.txt
timeout 300 python tools/prof_encode.py --n 1000000 --D 512 --d 128 --C 1 > $OUT/enc_cfg2.log 2>&1; tail -1 $OUT/enc_cfg2.log
timeout 300 python tools/prof_encode.py --n 1000000 --D 512 --d 96 --C 16 > $OUT/enc_cfg3.log 2>&1; tail -1 $OUT/enc_cfg3.log
timeout 300 python tools/prof_encode.py --n 4000000 --D 768 --d 160 --C 32 --xf16 > $OUT/enc_cfg5.log 2>&1; tail -1 $OUT/enc_cfg5.log
LV_K6_HPLANES=3 timeout 300 python tools/prof_encode.py --n 4000000 --D 768 --d 160 --C 32 --xf16 > $OUT/enc_cfg5_h3.log 2>&1; tail -1 $OUT/enc_cfg5_h3.log
LV_K6_DIRECT=0 timeout 300 python tools/prof_encode.py --n 4000000 --D 768 --d 160 --C 32 --xf16 > $OUT/enc_cfg5_bf16planes.log 2>&1; tail -1 $OUT/enc_cfg5_bf16planes.log
timeout 300 python tools/prof_encode.py --n 4000000 --D 200 --d 64 --C 1 --low fp16 > $OUT/enc_cfg4.log 2>&1; tail -1 $OUT/enc_cfg4.log
