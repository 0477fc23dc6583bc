import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
rng = np.random.default_rng(0)
for d in (200, 1000):
    S = rng.standard_normal((d, d))
    for n in (40, 41, 80, 81, 82):
        Y = rng.standard_normal((d, n))
        out = capi.tucker_debug_product(S, Y, 12345.0)
        print("d=%d n=%d  max |P1 - P2| = %.3e" % (d, n, out[0, 0]))
