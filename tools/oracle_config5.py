"""Offline fp64 oracle run of BASELINE.json config 5 (HOOI, 5 sweeps) -> a cache
the GPU parity test compares against ("If a full config-5 ...
oracle run is infeasible inside the benchmark, run it once offline and cache it").

Imports only synth/ (the seeded inputs) and oracle/ (the arithmetic).  Output:
tests/golden/config5_hooi_oracle.npz with the final factors (fp32; their rounding
moves the projector distance by ~1e-7, far below the 1e-4 bar), the core (fp64),
the per-sweep fits and the per-mode eigenvalue diagnostics (kappa, relative gap).

    python tools/oracle_config5.py [--sweeps 5] [--out tests/golden/config5_hooi_oracle.npz]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import tucker_oracle as O  # noqa: E402
from synth import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweeps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "config5_hooi_oracle.npz"))
    args = ap.parse_args()
    t0 = time.time()

    def log(msg):
        print(f"[{time.time() - t0:8.1f} s] {msg}", flush=True)

    c = make_config(5)
    log(f"config 5 generated: dims {c['dims']}, nnz {c['nnz']}, core {c['core']}")
    T = O.SparseTensor(c["dims"], c["idx"], c["vals"])
    del c["idx"], c["vals"]
    diag = []
    out = O.run_hooi_large(T, c["U0"], c["core"], args.sweeps, diag=diag, log=log)
    log("done")
    meta = dict(config=5, sweeps=args.sweeps, dims=list(c["dims"]), core=list(c["core"]), nnz=int(T.vals.size),
                seconds=time.time() - t0, cores=len(os.sched_getaffinity(0)),
                script="tools/oracle_config5.py (imports synth/ and oracle/ only)")
    np.savez(args.out, U_mode1=out["U"][0].astype(np.float32), U_mode2=out["U"][1].astype(np.float32),
             U_mode3=out["U"][2].astype(np.float32), G=out["G"], fits=np.asarray(out["fits"]),
             diag=json.dumps(diag), meta=json.dumps(meta))
    log(f"wrote {args.out}")
    for d in diag:
        print(json.dumps(d))


if __name__ == "__main__":
    main()
