# one full ncu capture of K6 at the cfg 2 shape (fp32 rows) and the cfg 5 shape (fp16 rows, 2M rows):
# raw metrics + per-source-line stall samples, summarised here (the .ncu-rep stays on the box)
OUT=gpurun_out/${OUTDIR:-k6ncu}
mkdir -p $OUT
cap() { name=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encode_tc -s 1 -c 1 -o /tmp/k6_$name python tools/prof_encode.py --reps 2 "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i /tmp/k6_$name.ncu-rep --page raw --csv > $OUT/raw_$name.csv 2>/dev/null
  ncu -i /tmp/k6_$name.ncu-rep --page source --csv > $OUT/source_$name.csv 2>/dev/null
  ls -la $OUT/raw_$name.csv $OUT/source_$name.csv; rm -f /tmp/k6_$name.ncu-rep; }
cap cfg2 --n 1000000 --D 512 --d 128 --C 1
cap cfg5 --n 2000000 --D 768 --d 160 --C 32 --xf16
