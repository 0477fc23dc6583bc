"""Check the fused eigensolver's k x k device routines against numpy (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
rng = np.random.default_rng(0)
for k in (5, 13, 40, 81, 82, 116):
    Y = rng.standard_normal((3 * k, k)) @ np.diag(np.logspace(0, 3, k))
    G = Y.T @ Y
    M = capi.tucker_debug_smalldense(0, G)
    I = M.T @ G @ M
    print("cholqr k=%3d  |M^T G M - I| = %.2e  upper=%s" % (k, np.abs(I - np.eye(k)).max(), np.allclose(np.tril(M, -1), 0)))
    Q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    w = np.sort(rng.uniform(1, 2, k))[::-1]
    H = (Q * w) @ Q.T
    for sw in (2, 3, 30):
        V, th, used = capi.tucker_debug_smalldense(1, H, max_sweeps=sw)
        off = V.T @ H @ V
        offn = np.linalg.norm(off - np.diag(np.diag(off))) / np.linalg.norm(H)
        print("  jacobi k=%3d sweeps<=%2d used %2d  offdiag %.2e  |VtV-I| %.2e  theta err %.2e" % (
            k, sw, used, offn, np.abs(V.T @ V - np.eye(k)).max(), np.abs(th - w).max()))
bad = 0
for d in (37, 200, 1000, 2000):
    S = rng.standard_normal((d, d))
    for n in range(1, 117):
        Y = rng.standard_normal((d, n)); D = rng.standard_normal((d, n))
        out = capi.tucker_debug_product(S, Y, 0.7, -0.3, D)
        ref = 0.7 * S @ Y - 0.3 * D
        err = np.abs(out - ref).max() / np.abs(ref).max()
        if not err < 1e-13:
            bad += 1
            print("PRODUCT MISMATCH d=%d n=%d err=%.2e" % (d, n, err))
print("product checks done, bad =", bad)
