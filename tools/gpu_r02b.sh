set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_memo.py tests/test_gpu_parity.py -m gpu -x -q -k "memo or order4 or end_to_end or determinism" > gpurun_out/memo_tests.log 2>&1; echo "rc=$?" >> gpurun_out/memo_tests.log
B="python bench.py --no-cpu-baseline --spttmc-configs="
timeout 600 $B > gpurun_out/bench_new.log 2>&1
TUCKER_EIG_EXCL=0 timeout 600 $B > gpurun_out/bench_noexcl.log 2>&1
TUCKER_HOOI_MEMO=0 timeout 600 $B > gpurun_out/bench_nomemo.log 2>&1
timeout 300 python tools/mp_timeline.py 4 > gpurun_out/mp_timeline.log 2>&1
TUCKER_EIG_EXCL=0 timeout 300 python tools/mp_timeline.py 4 > gpurun_out/mp_timeline_noexcl.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 --spttmc-configs=4 > gpurun_out/bench_tab4.log 2>&1
echo done
