set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/ttmc_time.py 3 5 > gpurun_out/ttmc3.log 2>&1
timeout 300 python tools/ttmc_time.py 1 5 > gpurun_out/ttmc1.log 2>&1
timeout 300 python tools/ttmc_time.py 2 5 > gpurun_out/ttmc2.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --spttmc-configs=1,2,3,4 > gpurun_out/bench_small.log 2>&1
echo done
