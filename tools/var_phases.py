"""Dev: fused-kernel phase timer of a variant build: python tools/var_phases.py <package root>."""
import os
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_12083_b200 as pkg

assert pkg.__file__.startswith(os.path.abspath(root)), pkg.__file__
from tools.probe_fused import plain, profile

plain(dict(rod_count=1, nodes_per_rod=100), steps=20000, cluster=16)
profile(dict(rod_count=1, nodes_per_rod=100), cluster=16)
