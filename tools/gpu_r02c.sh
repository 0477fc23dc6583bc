# round-2 late GPU run: parity suite, bench line, launch list, ncu full captures (args: what to run)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --spttmc-configs="
for w in "$@"; do
case $w in
tests) timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log ;;
smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log ;;
bench) timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
ref) timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log ;;
launches) timeout 600 $B > gpurun_out/b1.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1 ;;
ncu4) timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spttmc4_sib|k_spttmc4g<" -s 4 -c 2 -o gpurun_out/prof_ttmc4 python tools/ttmc_time.py 4 2 > gpurun_out/ncu_ttmc4.log 2>&1 ;;
ncuspmm) timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_w -s 30 -c 1 -o gpurun_out/prof_spmm $B > gpurun_out/ncu_spmm.log 2>&1 ;;
ncu3) timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spttmc3 -s 0 -c 6 -o gpurun_out/prof_ttmc3 python tools/ttmc_time.py 3 1 > gpurun_out/ncu_ttmc3.log 2>&1 ;;
esac
done
echo done
