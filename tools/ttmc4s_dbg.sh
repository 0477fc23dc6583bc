# k_spttmc4s phase-skipping timings (wrong results; timing only) -> gpurun_out/dbg.log
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in ${DBGS:-0 15 7}; do echo "dbg $d" >> gpurun_out/dbg.log; TUCKER_TTMC4=s TUCKER_TTMC4_DBG=$d python tools/ttmc_time.py 4 20 2>&1 | grep "mode 1" >> gpurun_out/dbg.log; done
TUCKER_TTMC4=g python tools/ttmc_time.py 4 20 2>&1 | grep "mode 1" | sed 's/^/g: /' >> gpurun_out/dbg.log
