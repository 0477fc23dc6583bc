python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sp.py tests/test_gpu_multigpu.py -x -q -k "gram or end_to_end or config1 or edge or world or sp" > gpurun_out/tq.log 2>&1; echo rc=$? >> gpurun_out/tq.log
timeout 300 python tools/mp_prof.py 4 3 > gpurun_out/mp4.log 2>&1
for o in 0 20 40 60 96; do echo "== OVS $o"; OVS=$o timeout 300 python tools/probe.py 4 5 2>&1 | grep -E "fits|^ \[\[|^ \[" ; done > gpurun_out/ovs.txt 2>&1
