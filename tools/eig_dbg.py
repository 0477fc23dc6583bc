import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__; __graft_entry__.build()
from paper_0711_2023_b200 import capi
from oracle import tucker_oracle as O
d, J, gap = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
rng = np.random.default_rng(d + J)
Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy(); w[0] = 60.0
w[J - 1] = w[J] * (1 + gap); w[:J] = np.maximum(w[:J], w[J - 1])
S = (Q * w) @ Q.T
dims, core = (8, 8, 8), (2, 2, 2)
r = np.random.default_rng(1)
from synth import uniform_distinct_coo, random_orthonormal
idx, vals = uniform_distinct_coo(dims, 50, r)
U0 = [random_orthonormal(8, 2, r) for _ in range(3)]
with capi.Tucker(dims, core, idx, vals, U0) as t:
    U, ev, rc = t.debug_eig(S, J)
    print("rc", rc, "stats", t.stats())
Uo, wo = O.leading_eigenvectors(S, J)
print("proj", O.projector_distance(U, Uo))
