# round evidence run: GPU suite, bench line, ncu launch list, full captures of the main kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
[ -z "$SKIP_TESTS" ] && { timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log; }
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --spttmc-configs="
timeout 600 $B > gpurun_out/b1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
for k in ${NCU_KERNELS:-k_eig_direct k_eig_fused k_spttmc4g k_spmm_w k_syrk_tc}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" -s ${NCU_SKIP:-6} -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
done
echo done
