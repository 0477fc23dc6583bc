set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/ttmc_time.py 3 5 > gpurun_out/ttmc3.log 2>&1
timeout 300 python tools/ttmc_time.py 1 5 > gpurun_out/ttmc1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hosvd.py tests/test_gpu_sp.py tests/test_gpu_multigpu.py tests/test_gpu_memo.py -m gpu -x -q > gpurun_out/gpu_tests_part.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_part.log
echo done
