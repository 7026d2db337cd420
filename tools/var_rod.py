"""Dev: rod-side HBM kernels of a variant build: python tools/var_rod.py <package root>."""
import json
import os
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_12083_b200 as pkg

assert pkg.__file__.startswith(os.path.abspath(root)), pkg.__file__
from tools.probe_rod import hbm_kernels

print(root, json.dumps({k: round(v["GB_per_s"]) for k, v in hbm_kernels().items()}))
