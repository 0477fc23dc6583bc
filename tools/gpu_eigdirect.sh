# direct eigensolver iteration: unit tests, per-phase times (tiled vs packed), host-timed solves
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_eig_units.py -x -q -rs -k small_dense > gpurun_out/ed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ed_tests.log
for d in 100 200 208; do
  TUCKER_EIG_PROF=1 timeout 120 python tools/eig_small_time.py $d 20 3 >> gpurun_out/ed_prof.log 2>&1
  TUCKER_EIG_PROF=1 TUCKER_EIG_DIRECT_OLD=1 timeout 120 python tools/eig_small_time.py $d 20 3 >> gpurun_out/ed_prof.log 2>&1
done
TAG=tiled timeout 120 python tools/eig_small_time.py 200 20 50 >> gpurun_out/ed_time.log 2>&1
TAG=packed TUCKER_EIG_DIRECT_OLD=1 timeout 120 python tools/eig_small_time.py 200 20 50 >> gpurun_out/ed_time.log 2>&1
[ -n "$BENCH" ] && { timeout 900 python bench.py $BENCH > gpurun_out/ed_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ed_bench.log; }
echo done
