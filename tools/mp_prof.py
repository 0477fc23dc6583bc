"""MP sweep of a BASELINE config (for ncu captures of k_spmm_mp / k_syrk_tc).
    python tools/mp_prof.py 4 [sweeps]"""
import sys
import torch
sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_0711_2023_b200 import capi  # noqa: E402
from synth import make_config  # noqa: E402

k = int(sys.argv[1])
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = make_config(k)
dev = torch.device("cuda", 0)
h = capi.tucker_init(c["dims"], c["core"], [torch.from_numpy(a).to(dev) for a in c["idx"]],
                     torch.from_numpy(c["vals"]).to(dev), [torch.from_numpy(u).to(dev) for u in c["U0"]],
                     on_device=True)
fits, stage, rc = capi.mp_sweep(h, sw, want_stage=True)
print(fits, stage)
capi.tucker_free(h)
