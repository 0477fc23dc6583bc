"""One-line summary of a bench.py JSON line on stdin (ms/step, sweeps, stage ms)."""
import json
import sys
d = json.loads(sys.stdin.read())
print(round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["sweep_ms"].items()},
      {k: round(v, 2) for k, v in d["roofline"]["stage_ms_per_step"].items()})
