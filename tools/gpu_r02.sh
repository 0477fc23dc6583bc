# round-2 GPU run: peaks, parity tests, bench line, launch list (args: what to run)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in "$@"; do
case $w in
peaks) timeout 300 python tools/peaks.py gpurun_out/measured_compute_peaks.json > gpurun_out/peaks.log 2>&1 ;;
tests) timeout 1800 python -m pytest tests -m gpu -x -q -s -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log ;;
quick) timeout 900 python -m pytest tests -m gpu -x -q -k "not config_full and not config5" > gpurun_out/gpu_quick.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_quick.log ;;
bench) timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
launches)
  B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --spttmc-configs="
  timeout 600 $B > gpurun_out/b1.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1 ;;
esac
done
echo done
