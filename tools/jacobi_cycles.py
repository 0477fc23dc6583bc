import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
rng = np.random.default_rng(0)
for k in (40, 60, 82, 116):
    Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    H = (Q * np.sort(rng.uniform(1, 2, k))[::-1]) @ Q.T
    for mode in (1, 2):
      V, th, used = capi.tucker_debug_smalldense(mode, H, max_sweeps=3)
      c = capi.tucker_debug_smalldense.cycles
      r = max(c[5], 1)
      print("mode %d " % mode + "k=%3d sweeps=%d rounds=%d per-round cycles: rot %.0f update %.0f | total %.0f cyc = %.1f us" % (
        k, used, c[5], c[0] / r, c[1] / r, c[6], c[6] / 1.9e3))
