"""Time the HOOI SpTTMc of every mode of a BASELINE config (tucker_time_ttmc) and
check one mode's Y against the fp64 oracle on sampled rows.
    python tools/ttmc_time.py 4 [reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import make_config  # noqa: E402

k = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
import __graft_entry__  # noqa: E402
__graft_entry__.build()
c = make_config(k, device="cuda" if k == 5 else None)
dev = torch.device("cuda", 0)
h = capi.tucker_init(c["dims"], c["core"], [torch.from_numpy(a).to(dev) for a in c["idx"]],
                     torch.from_numpy(c["vals"]).to(dev), [torch.from_numpy(u).to(dev) for u in c["U0"]],
                     on_device=True)
for n in range(len(c["dims"])):
    ms = capi.tucker_time_ttmc(h, n, reps)
    print(f"config {k} mode {n + 1}: {ms * 1e3:.1f} us", flush=True)
capi.tucker_free(h)
