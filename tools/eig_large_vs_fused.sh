python -c "import __graft_entry__ as g; g.build()"
for v in 0 1; do echo "== EIG_LARGE $v"; if [ $v = 1 ]; then export TUCKER_EIG_LARGE=1; fi; timeout 600 python tools/probe.py 4 5 2>&1 | grep -E "fits|^ \[\[|^ \[|eig_matvec" ; done
