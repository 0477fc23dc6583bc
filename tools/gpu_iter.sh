# iteration run: targeted GPU tests ($TESTS, a pytest -k expression), timings, bench line, optional ncu captures ($NCU: kernel regexes)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q -rs -k "$TESTS" > gpurun_out/it_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/it_tests.log; fi
if [ -n "$TTMC" ]; then
  for c in $TTMC; do timeout 300 python tools/ttmc_time.py $c 20 >> gpurun_out/it_ttmc.log 2>&1; TUCKER_TTMC4=g timeout 300 python tools/ttmc_time.py $c 20 | sed "s/^/g: /" >> gpurun_out/it_ttmc.log 2>&1; TUCKER_TTMC4=s timeout 300 python tools/ttmc_time.py $c 20 | sed "s/^/s: /" >> gpurun_out/it_ttmc.log 2>&1; done
fi
[ -n "$MICRO" ] && ./tools/lds_uniform_bench > gpurun_out/it_micro.log 2>&1
if [ -n "$BENCH" ]; then timeout 900 python bench.py $BENCH > gpurun_out/it_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/it_bench.log; fi
for k in $NCU; do
  kn=${k//[^a-zA-Z0-9_]/}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/it_$kn python bench.py --steps 1 --warmup 1 --no-cpu-baseline --spttmc-configs= > gpurun_out/it_ncu_$kn.log 2>&1
done
echo done
