for c in ${CFGS:-3 4 5}; do
  echo "== cfg $c"; free -g | sed -n 2p
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo rc=$?
  tail -4 gpurun_out/bench_cfg$c.err; cut -c1-900 gpurun_out/bench_cfg$c.json
done
