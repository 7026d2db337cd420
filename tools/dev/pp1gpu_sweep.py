import sys, os, json
sys.path.insert(0, '.')
import bench
from paper_2604_12083_b200.scenario import ScenarioConfig, build_initial_state, make_scenario
sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=100))
x0 = build_initial_state(sc)
r = bench.parareal_1gpu_leg(sc, x0, 0)
print(os.environ.get("PSWIM_ENGINE_FINE_CLUSTER"), os.environ.get("PSWIM_ENGINE_WAVE_CLUSTER"), round(r['serial_fine_steps_per_s']), round(r['l1']['value']), round(r['l1']['speedup_vs_serial_fine'],2), round(r['l2']['value']), round(r['l2']['speedup_vs_serial_fine'],2), r['l2']['eta'])
