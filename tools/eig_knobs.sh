# eigensolver knob sweep on config 2 (development aid): total eig ms over 5 HOOI + 5 MP sweeps
for o in 6 10 16; do for j in 1 2 3; do
  r=$(OVS=$o TUCKER_EIG_JSW=$j timeout 120 python tools/probe.py 2 5 2>&1 | python -c "
import sys, re, numpy as np
txt = sys.stdin.read()
tot = 0.0
for blk in re.findall(r'\[\[(.*?)\]\]', txt, re.S):
    rows = [list(map(float, l.replace('[','').replace(']','').split())) for l in blk.strip().split('\n')]
    tot += sum(r[2] for r in rows)
print('%.2f' % tot)")
  echo "ovs=$o jsw=$j eig_ms=$r"
done; done
