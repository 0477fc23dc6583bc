# SpTTMc per-launch times (config 2 probe, config 5 one sweep) -> gpurun_out/
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:spttmc --log-file gpurun_out/c2_ttmc.csv python tools/probe.py 2 1 > /dev/null 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:spttmc --log-file gpurun_out/c4_ttmc.csv python tools/probe.py 4 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:spttmc --log-file gpurun_out/c5_ttmc.csv python tools/config5.py 1 > /dev/null 2>&1
