"""Config 5 feasibility / timing probe (HOOI only; development aid).

Generates BASELINE.json config 5 (50000 x 50000 x 5000, 2e8 Zipf nonzeros),
builds the handle and runs HOOI sweeps, printing per-stage times and fits.
"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0711_2023_b200 import capi
from synth import make_config

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nnz = int(float(sys.argv[2])) if len(sys.argv) > 2 else None
t0 = time.time()
c = make_config(5, nnz=nnz, device="cuda")
print("gen %.1fs nnz %d" % (time.time() - t0, c["vals"].size), flush=True)
import resource
print("maxrss GB %.1f" % (resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6), flush=True)
t0 = time.time()
t = capi.Tucker(c["dims"], c["core"], c["idx"], c["vals"], c["U0"])
print("init %.2fs" % (time.time() - t0), flush=True)
del c["idx"]
t.stats(reset=True)
t0 = time.time()
fits, stage, rc = t.hooi_sweep(sweeps, want_stage=True)
print("hooi wall %.3fs rc %s fits %s" % (time.time() - t0, rc, fits), flush=True)
print("  stage ms [proj, gram, eig, core]:\n", stage)
print("  stats", t.stats(), flush=True)
t.close()
