"""One MP Gram (config 2, mode 0) through the debug entry point, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
from synth import make_config
c = make_config(2)
t = capi.Tucker(c["dims"], c["core"], c["idx"], c["vals"], c["U0"])
for _ in range(2):
    M = t.debug_gram(1, 0)
print(M[0, 0])
t.close()
