"""Check the torch-device Zipf generator reproduces the numpy one."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth.generators as G
for dims, nnz, batch in (((50, 60, 7), 2000, 1 << 10), ((50000, 50000, 5000), 3_000_000, 1 << 21)):
    a = G.zipf_coo(dims, nnz, np.random.default_rng(5), batch=batch)
    b = G.zipf_coo(dims, nnz, np.random.default_rng(5), batch=batch, device="cuda")
    print(dims, nnz, all(np.array_equal(x, y) for x, y in zip(a[0], b[0])), np.array_equal(a[1], b[1]))
t = time.time(); c = G.make_config(5, device="cuda"); print("config5 gen %.1fs" % (time.time() - t), c["vals"].size)
