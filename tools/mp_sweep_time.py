"""Per-sweep MP times at a config (repeated), for variance checks.   python tools/mp_sweep_time.py 2 [sweeps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import make_config  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = make_config(k)
dev = torch.device("cuda", 0)
h = capi.tucker_init(c["dims"], c["core"], [torch.from_numpy(a).to(dev) for a in c["idx"]],
                     torch.from_numpy(c["vals"]).to(dev), [torch.from_numpy(u).to(dev) for u in c["U0"]],
                     on_device=True)
out = []
for it in range(ns):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, st, _ = capi.mp_sweep(h, 1, want_stage=True)
    torch.cuda.synchronize()
    out.append((round(1e3 * (time.perf_counter() - t0), 2), [round(float(x), 2) for x in st[0]]))
print(f"config {k} MP sweeps (ms, stage ms proj/gram/eig/core):", out, flush=True)
capi.tucker_free(h)
