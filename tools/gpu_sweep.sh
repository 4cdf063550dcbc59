# bench line per config (full sizes); 10M configs use a smaller oracle sample
for c in ${CFGS:-1 2 3 4 5}; do
  oq=30; [ $c -ge 4 ] && oq=8
  timeout 1800 python bench.py --config $c --steps 20 --warmup 3 --oracle-queries $oq > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg $c rc=$?"; tail -2 gpurun_out/bench_cfg$c.err
done
# cfg 4's in-distribution family (its own fit and encode)
if [ -z "$CFGS" ] || [ -n "$CFG4_ID" ]; then
  timeout 1800 python bench.py --config 4 --family id --steps 20 --warmup 3 --oracle-queries 8 > gpurun_out/bench_cfg4id.json 2> gpurun_out/bench_cfg4id.err
  echo "cfg 4 id rc=$?"; tail -2 gpurun_out/bench_cfg4id.err
fi
