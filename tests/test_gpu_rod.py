"""GPU parity of the rotation square root and the rod load kernels (reference
rotation.cpp:91-107, rod.cpp:36-174) against the oracle and the reference's test bounds."""
import numpy as np
import pytest

from helpers import perturbed_rod, raw_rodrigues, rel_field_err

pytestmark = pytest.mark.gpu


def test_sqrt_rotation_matches_oracle_all_branches(gpu, oracle):
    from paper_2604_12083_b200.rotation import sqrt_rotation

    rng = np.random.default_rng(11)
    mats = []
    for i in range(3000):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        kind = i % 5
        th = {0: rng.uniform(0, np.pi), 1: rng.uniform(0, 1e-7), 2: np.pi - rng.uniform(0, 1e-2),
              3: np.pi - rng.uniform(0, 1e-6), 4: rng.uniform(1e-7, 1e-3)}[kind]
        mats.append(raw_rodrigues(ax, th))
    for ax in np.eye(3):
        mats.append(raw_rodrigues(ax, np.pi))
    mats.append(np.eye(3))
    mats = np.array(mats)
    got = sqrt_rotation(mats)
    want = np.array([oracle.sqrt_rotation(m) for m in mats])
    assert np.max(np.abs(got - want)) < 1e-12
    res = np.linalg.norm(got @ got - mats, axis=(1, 2))
    assert res.max() < 1e-7


def test_sqrt_rotation_paper_sampling_scheme(gpu, oracle):
    """test_rotation.cpp:88-114 statistics (mean <= 1e-13, max <= 1e-7, residual < 1e-12)."""
    from paper_2604_12083_b200.rotation import sqrt_rotation

    rng = np.random.default_rng(2024)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    rs = []
    for _ in range(100):
        th = rng.uniform(-0.1, np.pi + 0.1)
        n = axis
        if th < 0:
            n, th = -n, -th
        elif th > np.pi:
            n, th = -n, 2 * np.pi - th
        rs.append(raw_rodrigues(n, th))
    rs = np.array(rs)
    s = sqrt_rotation(rs)
    res = np.linalg.norm(s @ s - rs, axis=(1, 2))
    assert res.mean() <= 1e-13 and res.max() <= 1e-7
    for m in s:
        assert oracle.rotation_residual(m) < 1e-12


def test_sqrt_rotation_branch_continuity(gpu):
    """test_rotation.cpp:133-150: residual does not jump > 10x across either threshold."""
    from paper_2604_12083_b200.rotation import sqrt_rotation

    n = np.array([0.3, -0.5, 0.81])
    n /= np.linalg.norm(n)
    for pivot in (1e-7, np.pi - 1e-2):
        lo = [raw_rodrigues(n, pivot * (1 - 1e-3 * i)) for i in range(1, 9)]
        hi = [raw_rodrigues(n, pivot * (1 + 1e-3 * i)) for i in range(1, 9)]
        sl, sh = sqrt_rotation(np.array(lo)), sqrt_rotation(np.array(hi))
        rl = max(np.linalg.norm(a @ a - b) + 1e-16 for a, b in zip(sl, lo))
        rh = max(np.linalg.norm(a @ a - b) + 1e-16 for a, b in zip(sh, hi))
        assert max(rl / rh, rh / rl) < 10.0


@pytest.mark.parametrize("rods,m", [(1, 9), (3, 16), (5, 256), (2, 300)])
def test_rod_loads_match_oracle(gpu, oracle, rods, m):
    from paper_2604_12083_b200.rod import rod_loads
    from paper_2604_12083_b200.scenario import MaterialParams, ScenarioConfig, WaveformParams, make_scenario

    rng = np.random.default_rng(rods * 1000 + m)
    cfg = ScenarioConfig(rod_count=rods, nodes_per_rod=m, material=MaterialParams(0.8, 0.8, 1.2, 3.0, 3.0, 5.0),
                         waveform=WaveformParams(0.2, 1.5, 1.0))
    sc = make_scenario(cfg)
    state = np.concatenate([perturbed_rod(oracle, m, 1.0, rng, 0.08, 0.25) + np.array([0, 3.0 * r, 0] + [0] * 9)
                            for r in range(rods)])
    f, n, sf, sn = rod_loads(state.reshape(-1), 0.3, sc)
    mat6 = [0.8, 0.8, 1.2, 3.0, 3.0, 5.0]
    wave3 = [0.2, 1.5, 1.0]
    for r in range(rods):
        rod = state[r * m:(r + 1) * m]
        fo, mo = oracle.internal_loads(rod, 1.0, mat6, wave3, 0.3)
        nf, nn = oracle.nodal_loads(rod, 1.0, fo, mo)
        assert rel_field_err((sf[r * (m - 1):(r + 1) * (m - 1)], sn[r * (m - 1):(r + 1) * (m - 1)]), (fo, mo)) < 1e-12
        assert rel_field_err((f[r * m:(r + 1) * m], n[r * m:(r + 1) * m]), (nf, nn)) < 1e-11


def test_rod_balance_and_degenerate(gpu, oracle):
    """Free-rod force/torque balance (test_rod.cpp:103-124) and the degenerate-segment
    error (test_rod.cpp:66-70)."""
    from paper_2604_12083_b200 import PswimError
    from paper_2604_12083_b200.rod import rod_loads
    from paper_2604_12083_b200.scenario import MaterialParams, ScenarioConfig, WaveformParams, make_scenario

    rng = np.random.default_rng(101)
    sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=16, material=MaterialParams(0.7, 0.7, 1.1, 2, 2, 4),
                                      waveform=WaveformParams(0.3, 2.0, 0.8)))
    ds = 1.0 / 15
    for _ in range(5):
        rod = perturbed_rod(oracle, 16, 1.0, rng, 0.05, 0.2)
        f, n, _, _ = rod_loads(rod.reshape(-1), 0.4, sc)
        net_f = (f * ds).sum(0)
        net_t = ((np.cross(rod[:, 0:3], f) + n) * ds).sum(0)
        scale = max(1.0, np.abs(f).max())
        assert np.linalg.norm(net_f) / scale < 1e-10
        assert np.linalg.norm(net_t) / scale < 1e-10
    rod = perturbed_rod(oracle, 16, 1.0, rng, 0.05, 0.2)
    rod[5, 0:3] = rod[4, 0:3]
    with pytest.raises(PswimError):
        rod_loads(rod.reshape(-1), 0.0, sc)


def test_lj_matches_oracle(gpu, oracle):
    from paper_2604_12083_b200.rod import lj_repulsion
    from paper_2604_12083_b200.scenario import RANDOM, ScenarioConfig, build_initial_state, make_scenario

    cfg = ScenarioConfig(rod_count=12, nodes_per_rod=51, placement=RANDOM, lj_well_depth=0.01, seed=3)
    sc = make_scenario(cfg)
    x = build_initial_state(sc)
    rng = np.random.default_rng(0)
    x = x.reshape(-1, 12)
    x[:, 0:3] += rng.normal(scale=0.05, size=(len(x), 3))  # bring some pairs inside the cutoff
    x = x.reshape(-1)
    got = lj_repulsion(x, sc)
    want = oracle.lj_repulsion(x, 12, 51, 0.01, sc.lj_sigma, sc.lj_self_exclusion)
    assert np.abs(want).max() > 0
    assert np.max(np.abs(got - want)) <= 1e-12 * np.abs(want).max()


def test_rod_energy_gradient_and_objectivity(gpu, oracle):
    """test_rod.cpp:126-182 / acceptance C8 on the GPU loads: f = -dE/dx by central differences
    of the reference's discrete elastic energy (< 1e-6), and frame objectivity under a global
    rotation (< 1e-10)."""
    from paper_2604_12083_b200.rod import rod_loads
    from paper_2604_12083_b200.scenario import MaterialParams, ScenarioConfig, WaveformParams, make_scenario

    mat6 = [0.8, 0.8, 1.2, 3.0, 3.0, 5.0]
    wave3 = [0.2, 1.5, 1.0]
    sc = make_scenario(ScenarioConfig(rod_count=1, nodes_per_rod=9, material=MaterialParams(*mat6),
                                      waveform=WaveformParams(*wave3)))
    rng = np.random.default_rng(2023)
    ds = 1.0 / 8
    t = 0.25
    hstep = 3e-6 * ds
    for _ in range(5):
        rod = perturbed_rod(oracle, 9, 1.0, rng, 0.08, 0.25)
        f, n, _, _ = rod_loads(rod.reshape(-1), t, sc)
        scale = np.abs(f).max()
        worst = 0.0
        for k in range(9):
            for c in range(3):
                rp = rod.copy()
                rp[k, c] += hstep
                rm = rod.copy()
                rm[k, c] -= hstep
                want = -(oracle.elastic_energy(rp, 1.0, mat6, wave3, t) - oracle.elastic_energy(rm, 1.0, mat6, wave3, t)) / (2 * hstep * ds)
                worst = max(worst, abs(f[k, c] - want))
        assert worst / scale < 1e-6
        q = oracle.from_axis_angle(np.array([0.3, -0.4, 0.866]) / np.linalg.norm([0.3, -0.4, 0.866]), 1.234)
        rot = rod.copy()
        for blk in range(4):
            rot[:, 3 * blk:3 * blk + 3] = rod[:, 3 * blk:3 * blk + 3] @ q.T
        f2, n2, _, _ = rod_loads(rot.reshape(-1), t, sc)
        assert np.abs(f2 - f @ q.T).max() / scale < 1e-10
        assert np.abs(n2 - n @ q.T).max() / scale < 1e-10


def test_lj_pair_law_and_antisymmetry(gpu):
    """test_rod.cpp:184-254: LJ force vanishes at the cutoff, magnitude 24 w / sigma at r =
    sigma (repulsive), isolated pairs bitwise antisymmetric."""
    from paper_2604_12083_b200.rod import lj_repulsion
    from paper_2604_12083_b200.scenario import ScenarioConfig, make_scenario

    sigma, well = 0.5, 2.0
    sc = make_scenario(ScenarioConfig(rod_count=2, nodes_per_rod=3, rod_length=0.1, lj_well_depth=well,
                                      lj_sigma=sigma))

    def two_rods(d):
        x = np.zeros((6, 12))
        x[:, 3:6] = [0, 1, 0]
        x[:, 6:9] = [0, 0, 1]
        x[:, 9:12] = [1, 0, 0]
        for k in range(3):
            x[k, 0:3] = [k * 100.0, 0, 0]
            x[3 + k, 0:3] = [k * 100.0, d, 0]
        return x.reshape(-1)

    rc = 2 ** (1 / 6) * sigma
    assert np.all(lj_repulsion(two_rods(rc), sc) == 0.0)
    f = lj_repulsion(two_rods(sigma), sc)
    assert abs(np.linalg.norm(f[0]) - 24 * well / sigma) < 1e-12 * 24 * well / sigma
    assert f[0, 1] < 0
    f = lj_repulsion(two_rods(0.9 * sigma), sc)
    assert np.array_equal(f[0], -f[3])
