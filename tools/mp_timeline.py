"""MP sweep timeline at a BASELINE config (TUCKER_MP_TIMELINE=1): eigensolve end and the
side stream's SpMM / Gram end per mode, relative to the fork.   python tools/mp_timeline.py 4"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["TUCKER_MP_TIMELINE"] = "1"
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import make_config  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = make_config(k)
dev = torch.device("cuda", 0)
h = capi.tucker_init(c["dims"], c["core"], [torch.from_numpy(a).to(dev) for a in c["idx"]],
                     torch.from_numpy(c["vals"]).to(dev), [torch.from_numpy(u).to(dev) for u in c["U0"]],
                     on_device=True)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    capi.mp_sweep(h, 1)
    torch.cuda.synchronize()
    print(f"mp sweep {it}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
capi.tucker_free(h)
