mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_eig_units.py -x -q -rs -k small_dense > gpurun_out/ed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ed_tests.log
rm -f gpurun_out/ed_dbg.log
for dbg in 0 1 2; do TUCKER_EIG_DBG=$dbg TUCKER_EIG_PROF=1 timeout 120 python tools/eig_small_time.py 200 20 2 2>&1 | grep eig_direct_t | tail -1 | sed "s/^/dbg=$dbg /" >> gpurun_out/ed_dbg.log; done
TUCKER_EIG_DIRECT_OLD=1 TUCKER_EIG_PROF=1 timeout 120 python tools/eig_small_time.py 200 20 2 2>&1 | grep eig_direct | tail -1 >> gpurun_out/ed_dbg.log
TAG=tiled timeout 120 python tools/eig_small_time.py 200 20 50 >> gpurun_out/ed_dbg.log 2>&1
