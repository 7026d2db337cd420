"""Dev: phase timer of the 4 x 21 LJ system for a variant build: python tools/dev/var_ljphases.py <root>."""
import os
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2604_12083_b200 as pkg

assert pkg.__file__.startswith(os.path.abspath(root)), pkg.__file__
from tools.probe_fused import profile

profile(dict(rod_count=4, nodes_per_rod=21, placement=1, lj_well_depth=0.01, seed=2), cluster=4)
