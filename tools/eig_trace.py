"""Eigensolver trace on config-2 sweeps (development aid): per solve, outer
iterations and matvecs, for the current TUCKER_EIG path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
from synth import make_config
c = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t = capi.Tucker(c["dims"], c["core"], c["idx"], c["vals"], c["U0"])
for algo in ("hooi", "mp"):
    t.set_factors(c["U0"])
    for s in range(sw):
        t.stats(reset=True)
        f = getattr(t, algo + "_sweep")
        fits, stage, rc = f(1, want_stage=True) if algo == "hooi" else f(1, want_fit=True, want_stage=True)
        st = t.stats()
        print(algo, s, "rc", rc, "fit %.8f" % fits[0], "eig ms %.2f" % stage[0][2], "outer", st["eig_outer"],
              "matvec", st["eig_matvec"], "jsw", st["jacobi_sweeps"], flush=True)
t.close()
