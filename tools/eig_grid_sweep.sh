python -c "import __graft_entry__ as g; g.build()"
for g in 148 64 32 16 8; do
  TUCKER_EIG_GRID=$g timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --spttmc-configs= > gpurun_out/eg_$g.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/eg_$g.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print($g, d.get('ms_per_step'), d.get('roofline',{}).get('stage_ms_per_step'), d.get('fit'))
PY
done
