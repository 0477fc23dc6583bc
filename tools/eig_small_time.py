"""Time the dense eigensolvers on a d x d Gram-like matrix (flat bulk + top outliers, MP-like):
one-CTA k_eig_direct (default), the 4-CTA cluster path (TUCKER_EIG_CLUSTER=1) and the fused
iterative solver (TUCKER_EIG_FUSED=1).   python tools/eig_small_time.py [d] [J] [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import random_orthonormal, uniform_distinct_coo  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 200
J = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rng = np.random.default_rng(3)
Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
w = np.sort(rng.uniform(0.9, 1.0, d))[::-1].copy()
w[:J] = np.linspace(40, 1.05, J)
S = (Q * w) @ Q.T
dims, core = (8, 8, 8), (2, 2, 2)
idx, vals = uniform_distinct_coo(dims, 50, np.random.default_rng(1))
U0 = [random_orthonormal(I, c, np.random.default_rng(2)) for I, c in zip(dims, core)]
with capi.Tucker(dims, core, idx, vals, U0) as t:
    t.debug_eig(S, J)
    t0 = time.perf_counter()
    for _ in range(reps):
        t.debug_eig(S, J)
    print(f"{os.environ.get('TAG', 'default')}: d={d} J={J}: {1e3 * (time.perf_counter() - t0) / reps:.3f} ms per solve "
          f"(host-timed, incl. H2D of S and D2H)", flush=True)
