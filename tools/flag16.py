"""Dev: one fused flagellum launch (cluster 16, 2000 RK2 steps) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.probe_fused import plain

plain(dict(rod_count=1, nodes_per_rod=100), steps=int(sys.argv[1]) if len(sys.argv) > 1 else 2000)
