# eigensolver per-phase / per-product timers (development aid): build with
# TK_EIG_PROFILE=1, run tools/probe.py (config, sweeps), rebuild the default library
set -e
TUCKER_NVCC_EXTRA=-DTK_EIG_PROFILE=1 python -m paper_0711_2023_b200._build --force > /dev/null
timeout 300 python tools/probe.py ${1:-2} ${2:-5}
python -m paper_0711_2023_b200._build --force > /dev/null
