import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__
__graft_entry__.build()
from paper_0711_2023_b200 import capi
print(capi.tucker_debug_product_time(1000, 82, 10))
