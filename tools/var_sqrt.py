"""Dev: batched sqrt throughput of a variant build: python tools/var_sqrt.py <package root>."""
import os
import runpy
import sys

root = sys.argv[1]
sys.path.insert(0, root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_12083_b200 as pkg

assert pkg.__file__.startswith(os.path.abspath(root)), pkg.__file__
print(root, end=" ")
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe_sqrt.py"), run_name="__main__")
