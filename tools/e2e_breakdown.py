"""Where an e2e bench step's time goes: fresh handle from pinned host buffers
(init, HOOI sweeps, core, MP sweeps, core) vs the same sweeps on a reused handle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0711_2023_b200 import capi
from synth import make_config
c = make_config(2)
dims, core, S = c["dims"], c["core"], c["sweeps"]
idx_h = [torch.from_numpy(a).pin_memory() for a in c["idx"]]
vals_h = torch.from_numpy(c["vals"]).pin_memory()
U0_h = [torch.from_numpy(u).pin_memory() for u in c["U0"]]
st = torch.cuda.current_stream()
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = t(); h = capi.tucker_init(dims, core, [a.numpy() for a in idx_h], vals_h.numpy(), [u.numpy() for u in U0_h], stream=st.cuda_stream)
    t1 = t(); capi.hooi_sweep(h, S); t2 = t(); capi.core_and_fit(h, dims, core); t3 = t()
    capi.tucker_set_factors(h, [u.numpy() for u in U0_h]); t4 = t(); capi.mp_sweep(h, S, want_fit=False); t5 = t()
    capi.core_and_fit(h, dims, core); t6 = t()
    capi.tucker_set_factors(h, [u.numpy() for u in U0_h]); t7 = t(); capi.hooi_sweep(h, S); t8 = t()
    capi.tucker_set_factors(h, [u.numpy() for u in U0_h]); t9 = t(); capi.mp_sweep(h, S, want_fit=False); t10 = t()
    capi.tucker_free(h)
    print("init %.1f hooi %.1f core %.1f setf %.1f mp %.1f core %.1f | reused: hooi %.1f mp %.1f (ms)" % tuple(
        1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t8 - t7, t10 - t9)), flush=True)
