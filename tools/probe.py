"""Quick timing probe of the CUDA path on one config (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
from synth import make_config

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.time(); c = make_config(k); print("gen %.1fs" % (time.time() - t0), flush=True)
t0 = time.time()
t = capi.Tucker(c["dims"], c["core"], c["idx"], c["vals"], c["U0"], eig_oversample=int(os.environ.get("OVS", "0")))
print("init %.2fs" % (time.time() - t0), flush=True)
for algo in ("hooi", "mp"):
    t.set_factors(c["U0"]); t.stats(reset=True)
    t0 = time.time()
    f = getattr(t, algo + "_sweep")
    fits, stage, rc = f(sweeps, want_stage=True) if algo == "hooi" else f(sweeps, want_fit=True, want_stage=True)
    el = time.time() - t0
    print(algo, "wall %.3fs" % el, "rc", rc, "fits", fits)
    print("  stage ms [proj, gram, eig, core]:\n", stage)
    print("  stats", t.stats())
t.close()
