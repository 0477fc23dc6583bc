set -e
TUCKER_NVCC_EXTRA=-DTK_GSYNC_STATS=1 python -m paper_0711_2023_b200._build --force > /dev/null
TUCKER_EIG_DEBUG=1 timeout 300 python tools/eig_trace.py 2 3 > gpurun_out/gs.log 2>&1
python -m paper_0711_2023_b200._build --force > /dev/null
