import sys, json, types
sys.path.insert(0, '.')
import bench
from paper_2604_12083_b200 import _lib
args = types.SimpleNamespace(no_cpu=False)
leg = bench.flagellum_leg(args, 0, "cuda:0")
leg.pop("parareal_1gpu", None)
print(json.dumps(leg, indent=1, default=str))
