mkdir -p gpurun_out/r02i8
for spec in "5 --low i8" "2 --low i8" "1"; do
  name=$(echo "$spec" | tr -d ' -' )
  timeout 1200 python bench.py --config $spec --steps 20 --warmup 5 > gpurun_out/r02i8/bench_cfg$name.json 2> gpurun_out/r02i8/bench_cfg$name.err
  echo "cfg $spec rc=$?"
done
