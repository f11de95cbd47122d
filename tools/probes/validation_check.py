import sys
sys.path.insert(0, '.')
import paper_2501_07018_b200 as P
from tests.test_gpu_parity import _tamper
for kind in ["layout_index", "index_wraps", "index_huge", "index_negative", "start_wraps", "index_wraps_staged"]:
    p = _tamper(kind)
    try:
        P.solve(p)
        print(kind, "NO ERROR")
    except ValueError as e:
        print(kind, "->", e)
