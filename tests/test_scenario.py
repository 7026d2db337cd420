"""Native scenario construction == the reference's (scenario.cpp:10-120), bitwise (no GPU)."""
import numpy as np
import pytest

from oracle.pyoracle import Scenario as OS
from paper_2604_12083_b200.scenario import RANDOM, ScenarioConfig, build_initial_state, make_scenario


@pytest.mark.parametrize("kw", [dict(rod_count=1, nodes_per_rod=21), dict(rod_count=64, nodes_per_rod=256, epsilon=0.08),
                                dict(rod_count=7, nodes_per_rod=33, placement=RANDOM, seed=5),
                                dict(rod_count=12, nodes_per_rod=51, placement=RANDOM, lj_well_depth=0.01, seed=3)])
def test_initial_state_matches_oracle(oracle, kw):
    sc = make_scenario(ScenarioConfig(**kw))
    osc = OS.make(**kw)
    r = oracle.resolve(osc)
    assert sc.ds == r.ds and sc.epsilon == r.epsilon and sc.lj_sigma == r.lj_sigma
    assert sc.lj_self_exclusion == r.lj_self_exclusion
    assert np.array_equal(build_initial_state(sc), oracle.build_initial_state(osc))


def test_scenario_validation():
    from paper_2604_12083_b200 import InvalidArgument

    with pytest.raises(InvalidArgument):
        make_scenario(ScenarioConfig(nodes_per_rod=2))
    with pytest.raises(InvalidArgument):
        make_scenario(ScenarioConfig(rod_count=0))
    with pytest.raises(InvalidArgument):
        make_scenario(ScenarioConfig(mu=0.0))


def test_pack_unpack_and_metric(oracle):
    from paper_2604_12083_b200.io import pack_state, rod_position_metric, unpack_state

    sc = make_scenario(ScenarioConfig(rod_count=3, nodes_per_rod=5))
    x = build_initial_state(sc)
    u = unpack_state(x, 3, 5)
    assert np.array_equal(pack_state(u), x)
    assert np.array_equal(u[1, 2, 0], x[12 * 7:12 * 7 + 3])
    y = x + np.random.default_rng(0).normal(scale=1e-3, size=x.shape)
    assert rod_position_metric()(x, y) == oracle.position_metric(x, y)
