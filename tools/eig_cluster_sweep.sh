python -c "import __graft_entry__ as g; g.build()"
for cfg in 4 2; do for c in 0 8 16; do
  echo "== config $cfg cluster $c"
  TUCKER_EIG_CLUSTER=$c timeout 300 python tools/probe.py $cfg 5 2>&1 | grep -E "fits|eig_phase|^ \[\[|^ \[" | head -20
done; done
