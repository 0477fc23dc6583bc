# round-end style GPU run: parity tests, bench line, ncu launch list + full captures
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
[ -z "$SKIP_TESTS" ] && { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log; }
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eig_fused -s 40 -c 1 -o gpurun_out/prof_eig $B > gpurun_out/ncu_eig.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_syrk_tc -s 1 -c 1 -o gpurun_out/prof_gram_mp python tools/prof_gram.py > gpurun_out/ncu_gram.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spttmc3 -s 10 -c 1 -o gpurun_out/prof_spttmc $B > gpurun_out/ncu_spttmc.log 2>&1
echo done
