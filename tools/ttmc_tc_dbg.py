"""Compare the tcgen05 SpTTMc against the SIMT one (error pattern)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import uniform_distinct_coo, random_orthonormal
dims, core = (40, 30, 50), tuple(int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (10, 10, 10)))
rng = np.random.default_rng(1)
idx, vals = uniform_distinct_coo(dims, 3000, rng)
U0 = [random_orthonormal(I, J, np.random.default_rng(2 + n)) for n, (I, J) in enumerate(zip(dims, core))]
np.savez("/tmp/dbg_in.npz", *idx, vals, *U0)
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_0711_2023_b200 import capi
d = np.load("/tmp/dbg_in.npz"); a = [d["arr_" + str(i)] for i in range(7)]
t = capi.Tucker(DIMS, CORE, a[:3], a[3], a[4:7])
np.save(sys.argv[1], t.debug_ttmc(0)); t.close()
'''.replace("DIMS", repr(dims)).replace("CORE", repr(core))
for tag, env in (("tc", {}), ("simt", {"TUCKER_TTMC": "simt"})):
    subprocess.run([sys.executable, "-c", code, "/tmp/y_%s.npy" % tag], env={**os.environ, **env}, check=True)
Yt, Ys = np.load("/tmp/y_tc.npy"), np.load("/tmp/y_simt.npy")
print("rel err", np.linalg.norm(Yt - Ys) / np.linalg.norm(Ys))
J1, J2 = core[1], core[2]
# columns in Kolda order: (mode1 index fastest) -> reshape rows x J2 x J1
A = Yt.reshape(-1, J2, J1); B = Ys.reshape(-1, J2, J1)
print("row 0 tc:\n", np.round(A[0, :4, :6], 4)); print("row 0 simt:\n", np.round(B[0, :4, :6], 4))
print("ratio sample", np.round((A[0] / np.where(B[0] == 0, 1, B[0]))[:4, :6], 3))
