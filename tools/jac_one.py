"""One mode-2 Jacobi unit launch (k from argv) for ncu source-level profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0711_2023_b200 import capi
k = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(0)
Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
H = (Q * np.sort(rng.uniform(1, 2, k))[::-1]) @ Q.T
V, th, used = capi.tucker_debug_smalldense(2, H, max_sweeps=2)
print("used", used)
