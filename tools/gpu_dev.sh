# development GPU run: microbench, parity tests, probe
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && timeout 60 /tmp/mb > gpurun_out/mb.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/t_gpu.log
timeout 300 python tools/probe.py 2 5 > gpurun_out/probe_fused.log 2>&1; echo "rc=$?" >> gpurun_out/probe_fused.log
