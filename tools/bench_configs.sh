# bench.py at other BASELINE configs -> gpurun_out/bench_cfg.log
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CFGS:-2 3 1}; do
  echo "config $c" >> gpurun_out/bench_cfg.log
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --spttmc-configs= > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log | python tools/bench_brief.py >> gpurun_out/bench_cfg.log 2>&1
done
