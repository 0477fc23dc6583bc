"""Config-5 MP (sparse multislice Gram + large-d eigensolver): time `sweeps` MP sweeps.
    python tools/c5_mp.py [sweeps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import make_config  # noqa: E402

sw = int(sys.argv[1]) if len(sys.argv) > 1 else 1
t0 = time.time()
c = make_config(5, device="cuda")
print(f"gen {time.time() - t0:.1f} s", flush=True)
dev = torch.device("cuda", 0)
h = capi.tucker_init(c["dims"], c["core"], [torch.from_numpy(a).to(dev) for a in c["idx"]],
                     torch.from_numpy(c["vals"]).to(dev), [torch.from_numpy(u).to(dev) for u in c["U0"]],
                     on_device=True)
for s in range(sw):
    t0 = time.time()
    fits, stage, rc = capi.mp_sweep(h, 1, want_stage=True)
    print(f"MP sweep {s}: {time.time() - t0:.2f} s, rc {rc}, fit {fits[0]:.8f}, stage ms {stage[0]}, "
          f"stats {capi.tucker_stats(h, reset=True)['eig_matvec']} products", flush=True)
capi.tucker_free(h)
