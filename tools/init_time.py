"""tucker_init phase times (TUCKER_PROFILE_INIT) on config 2 from host buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TUCKER_PROFILE_INIT"] = "1"
from paper_0711_2023_b200 import capi
from synth import make_config
c = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for rep in range(3):
    t0 = time.perf_counter()
    h = capi.tucker_init(c["dims"], c["core"], c["idx"], c["vals"], c["U0"])
    print("total %.2f ms" % ((time.perf_counter() - t0) * 1e3), file=sys.stderr, flush=True)
    capi.tucker_free(h)
