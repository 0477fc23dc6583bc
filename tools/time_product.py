import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
capi.tucker_debug_product_time(1000, 82, 5)  # warm-up
for d, n in [(1000, 82), (1000, 50), (1000, 34), (2000, 42), (200, 40), (5000, 116)]:
    us = capi.tucker_debug_product_time(d, n, 50)
    print("d=%5d n=%3d  %8.2f us  %.2f TFLOP/s" % (d, n, us, 2.0 * d * d * n / us / 1e6))
