"""GPU narrow phase vs the CPU oracle: bit-exact TOIs, hit sets and classes.

Bar (north star): CCD hit/miss sets must match bit-exactly given identical
positions; we require the stronger property that every fp64 output is
bitwise identical (NaN where the oracle has NaN).
"""

import numpy as np
import pytest

from oracle import narrow as O

pytestmark = pytest.mark.gpu


def _random_pairs(n, rng, spread=1.0, speed=1.0):
    """reference tests/test_ccd.py:53-59."""
    kind = np.zeros(n, dtype=np.int8)
    kind[n // 2:] = 1
    x0 = spread * rng.uniform(-1.0, 1.0, size=(4 * n, 3))
    x1 = x0 + speed * rng.uniform(-1.0, 1.0, size=(4 * n, 3))
    return kind, np.arange(4 * n).reshape(n, 4), x0, x1


def _near_contact_pairs(n, rng):
    """Pairs near grazing/coplanar configurations: the edge cases of the root finder."""
    kind = (rng.random(n) < 0.5).astype(np.int8)
    base = rng.normal(size=(n, 4, 3)) * 0.2
    base[:, :, 2] *= 1e-3 * rng.random((n, 1))           # nearly coplanar
    move = rng.normal(size=(n, 4, 3)) * 0.01
    move[rng.random(n) < 0.2] = 0.0                       # static pairs
    move[rng.random(n) < 0.2, :, 2] = 0.0                 # in-plane motion (flat cubic)
    x0 = base.reshape(-1, 3)
    x1 = (base + move).reshape(-1, 3)
    return kind, np.arange(4 * n).reshape(n, 4), x0, x1


def _same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(
        a[~np.isnan(a)].view(np.uint64), b[~np.isnan(b)].view(np.uint64))


def test_full_ccd_known_answers(cuda):
    import paper_2403_19272_b200 as P

    x0 = np.array([[0.25, 0.25, -1.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    x1 = x0.copy()
    x1[0, 2] = 1.0
    assert np.isclose(P.full_ccd(np.array([0]), np.array([[0, 1, 2, 3]]), x0, x1)[0], 0.5, atol=1e-9)
    assert np.isclose(P.global_toi(np.array([0]), np.array([[0, 1, 2, 3]]), x0, x1, alpha=0.8), 0.4)
    e0 = np.array([[-1.0, 0.0, -1.0], [1.0, 0.0, -1.0], [0.0, -1.0, 0.0], [0.0, 1.0, 0.0]])
    e1 = e0.copy()
    e1[:2, 2] = 1.0
    assert np.isclose(P.full_ccd(np.array([1]), np.array([[0, 1, 2, 3]]), e0, e1)[0], 0.5, atol=1e-9)
    # coplanar slide -> flat-cubic fallback (reference tests/test_ccd.py:144-154)
    s0 = np.array([[-2.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [1.0, 0.0, 0.0], [2.0, 0.0, 0.0]])
    s1 = s0.copy()
    s1[:2, 0] += 3.0
    t = P.full_ccd(np.array([1]), np.array([[0, 1, 2, 3]]), s0, s1)[0]
    assert abs(t - 2.0 / 3.0) <= 1.0 / 32.0
    # receding from touch is not an impact
    r0 = np.array([[0.25, 0.25, 0.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    r1 = r0.copy()
    r1[0, 2] = 1.0
    assert np.isnan(P.full_ccd(np.array([0]), np.array([[0, 1, 2, 3]]), r0, r1)[0])


@pytest.mark.parametrize("maker", [_random_pairs, _near_contact_pairs])
def test_full_ccd_bitwise_vs_oracle(cuda, rng, maker):
    import paper_2403_19272_b200 as P

    kind, idx, x0, x1 = maker(20000, rng)
    got = P.full_ccd(kind, idx, x0, x1)
    ref = O.full_ccd(kind, idx, x0, x1)
    assert _same(got, ref)
    assert (~np.isnan(ref)).sum() > 100


def test_full_ccd_single_pair_path(cuda, rng):
    """m == 1 uses OpenBLAS's other summation order (SURVEY.md section 7 hard part 1)."""
    import paper_2403_19272_b200 as P

    kind, idx, x0, x1 = _random_pairs(300, rng)
    for i in range(300):
        got = P.full_ccd(kind[i:i + 1], idx[i:i + 1] - 4 * i, x0[4 * i:4 * i + 4], x1[4 * i:4 * i + 4])
        ref = O.full_ccd(kind[i:i + 1], idx[i:i + 1] - 4 * i, x0[4 * i:4 * i + 4], x1[4 * i:4 * i + 4])
        assert _same(got, ref), i


@pytest.mark.parametrize("floor", [0.2, 1.0 - 0.8])
def test_distance_toi_bitwise(cuda, rng, floor):
    import paper_2403_19272_b200 as P

    for maker in (_random_pairs, _near_contact_pairs):
        kind, idx, x0, x1 = maker(20000, rng)
        got = P.distance_toi(kind, idx, x0, x1, floor_frac=floor)
        ref = O.distance_toi(kind, idx, x0, x1, floor_frac=floor)
        assert _same(got, ref)


def _comoving_pairs(n, rng, scale=0.002, shift=0.003, twist=0.02):
    """Pairs a few mm apart carried along by a common rigid motion (rotation about z
    + translation) plus a small relative jitter: the cloth-riding-the-body regime."""
    kind = (rng.random(n) < 0.5).astype(np.int8)
    c = rng.uniform(-0.3, 0.3, size=(n, 1, 3))
    base = c + rng.normal(size=(n, 4, 3)) * scale
    ang = twist * rng.uniform(0.5, 1.0, size=(n, 1))
    ca, sa = np.cos(ang), np.sin(ang)
    x, y = base[..., 0], base[..., 1]
    end = np.stack([ca * x - sa * y, sa * x + ca * y, base[..., 2]], axis=-1)
    end = end + shift * rng.normal(size=(n, 1, 3)) + 1e-5 * rng.normal(size=(n, 4, 3))
    return kind, np.arange(4 * n).reshape(n, 4), base.reshape(-1, 3), end.reshape(-1, 3)


@pytest.mark.parametrize("floor", [0.2, 0.5])
def test_distance_toi_comoving_bitwise(cuda, rng, floor):
    """Exercises the march's relative-motion shortcut (narrow.cu march_never_reaches):
    results must stay bitwise the oracle's, NaN or not."""
    import paper_2403_19272_b200 as P

    kind, idx, x0, x1 = _comoving_pairs(20000, rng)
    got = P.distance_toi(kind, idx, x0, x1, floor_frac=floor)
    ref = O.distance_toi(kind, idx, x0, x1, floor_frac=floor)
    assert np.isnan(ref).mean() > 0.3 and (~np.isnan(ref)).any()
    assert _same(got, ref)


@pytest.mark.parametrize("count", [1, 3, 6])
def test_partial_ccd_bitwise(cuda, rng, count):
    """reference tests/test_partial_ccd.py:68-88 population."""
    import paper_2403_19272_b200 as P

    m = 20000
    kind = np.zeros(m, dtype=np.int8)
    kind[m // 2:] = 1
    x0 = rng.normal(size=(4 * m, 3))
    x1 = x0 + 0.4 * rng.normal(size=(4 * m, 3))
    idx = np.arange(4 * m).reshape(m, 4)
    got = P.partial_ccd(kind, idx, x0, x1, P.default_samples(count))
    ref = O.partial_ccd(kind, idx, x0, x1, count)
    assert np.array_equal(got, ref)
    assert 0 < ref.sum() < m


def test_pair_witness_bitwise(cuda, rng):
    import paper_2403_19272_b200 as P

    kind, idx, x0, _ = _near_contact_pairs(20000, rng)
    got = P.pair_witness(kind, idx, x0)
    ref = O.witness(kind, idx, x0)
    for g, r in zip(got, ref):
        assert _same(g, r)


def test_pair_witness_degenerate(cuda):
    """Touching witnesses fall back to triangle normals / edge cross (stepper.py:201-213)."""
    from paper_2403_19272_b200.collision import witness_normals

    x = np.array([[0.2, 0.2, 0.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0],
                  [0.5, -1.0, 0.0], [0.5, 1.0, 0.0], [0.0, 0.5, 0.0], [1.0, 0.5, 0.0]])
    kind = np.array([0, 1], dtype=np.int8)
    idx = np.array([[0, 1, 2, 3], [4, 5, 6, 7]])
    bary, dist, nrm = witness_normals(kind, idx, x)
    assert dist.max() <= 1e-12
    assert np.allclose(np.abs(nrm[0]), [0, 0, 1]) and np.allclose(np.abs(nrm[1]), [0, 0, 1])
    from oracle.stepper import OracleSimulation, Pairs

    pr = Pairs(kind, idx)
    OracleSimulation.witness_into(None, pr, x)
    assert np.array_equal(nrm, pr.normal) and np.array_equal(bary, pr.bary) and np.array_equal(dist, pr.dist)


@pytest.mark.parametrize("steps,jitter,move", [(0, 0.0, 2e-3), (12, 0.0, 1e-3), (6, 2e-4, 5e-4), (3, 0.0, 0.0)])
def test_ccd_site_matches_oracle(cuda, rng, steps, jitter, move):
    """The step's CCD site (broad phase + filter/worklist narrow phase) returns, pair for
    pair, exactly the oracle's full_ccd and distance_toi values (bitwise, NaN-aware),
    including motion-free sites (exit line search) and grazing contact."""
    import paper_2403_19272_b200 as P
    from oracle import narrow

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    for _ in range(steps):
        sim.step()
    x0 = sim.world(sim.state.x)
    x0 = x0 + jitter * rng.normal(size=x0.shape)
    x1 = x0 + move * rng.normal(size=x0.shape)
    x1[len(sim.state.x):] = x0[len(sim.state.x):]
    pairs, toi, filt = sim._full_ccd_site(x0, x1)
    assert len(pairs) > 0
    ref_toi = narrow.full_ccd(pairs.kind, pairs.idx, x0, x1)
    ref_filt = narrow.distance_toi(pairs.kind, pairs.idx, x0, x1, floor_frac=1.0 - sim.config.alpha)
    assert _same(toi, ref_toi)
    assert _same(filt, ref_filt)
    if steps == 12 or move == 0.0:
        assert (~np.isnan(ref_filt)).any() or move == 0.0


@pytest.mark.parametrize("angle,shift", [(0.02, 0.003), (0.005, 0.0)])
def test_ccd_site_rigid_motion_matches_oracle(cuda, rng, angle, shift):
    """Site filter's relative-motion bound (the whole world riding a rigid motion, like
    the skirt on its spinning body): every pair's values still equal the oracle's."""
    import paper_2403_19272_b200 as P
    from oracle import narrow

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    for _ in range(12):
        sim.step()
    x0 = sim.world(sim.state.x)
    ca, sa = np.cos(angle), np.sin(angle)
    x1 = np.stack([ca * x0[:, 0] - sa * x0[:, 1], sa * x0[:, 0] + ca * x0[:, 1], x0[:, 2]], axis=1)
    x1 = x1 + shift + 2e-5 * rng.normal(size=x0.shape)
    pairs, toi, filt = sim._full_ccd_site(x0, x1)
    assert len(pairs) > 0
    ref_toi = narrow.full_ccd(pairs.kind, pairs.idx, x0, x1)
    ref_filt = narrow.distance_toi(pairs.kind, pairs.idx, x0, x1, floor_frac=1.0 - sim.config.alpha)
    assert _same(toi, ref_toi)
    assert _same(filt, ref_filt)
