# bench at several fused-eigensolver grid sizes (TUCKER_EIG_GRID) -> gpurun_out/grid.log
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for gsz in ${GRIDS:-32 16 8 64}; do
  TUCKER_EIG_GRID=$gsz python bench.py --steps 3 --warmup 3 --no-cpu-baseline --spttmc-configs= > gpurun_out/grid_$gsz.log 2>&1
  echo "grid $gsz" >> gpurun_out/grid.log
  tail -1 gpurun_out/grid_$gsz.log | python tools/bench_brief.py >> gpurun_out/grid.log 2>&1
done
