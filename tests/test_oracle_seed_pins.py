"""Pins of the initial-partition oracle (oracle/seed.py, X20-X23)
against hand values, closed forms and brute force — never against the oracle itself."""
import numpy as np
import pytest

from oracle import seed


def test_member_means_hand():
    off = np.array([0, 2, 3])
    Y = np.array([[0.0, 0.0], [2.0, 4.0], [-1.0, 5.0]])
    om = np.array([0.25, 0.75, 1.0])
    mu = seed.member_means(off, Y, om)
    assert np.array_equal(mu, [[1.5, 3.0], [-1.0, 5.0]])


def test_sq_dist_hand():
    assert np.array_equal(seed.sq_dist(np.array([[1.0, 2.0, 2.0], [0.0, 0.0, 3.0]]), np.zeros(3)), [9.0, 9.0])
    assert seed.sq_dist(np.array([[4.0, -1.0]]), np.array([1.0, 3.0]))[0] == 25.0


@pytest.mark.parametrize("u1, want", [(0.05, 1.0), (0.099, 1.0), (0.1, 3.0), (0.2, 3.0), (0.0, 1.0), (0.999, 3.0)])
def test_d2_seeding_inverse_cdf_hand(u1, want):
    # points 0, 1, 3; first centre u0 = 0 -> point 0; D^2 = 0, 1, 9 (sum 10): P(1) = 0.1, P(3) = 0.9.
    # The first index whose prefix (0, 1, 10) exceeds u1 * 10 (X20).
    P = np.array([[0.0], [1.0], [3.0]])
    c = seed.kmeanspp(P, 2, [0.0, u1], 0)
    assert c[0, 0] == 0.0 and c[1, 0] == want


def test_first_centre_is_floor_u_ns():
    P = np.arange(10.0)[:, None]
    for u0, want in ((0.0, 0.0), (0.35, 3.0), (0.999, 9.0)):
        assert seed.kmeanspp(P, 1, [u0], 0)[0, 0] == want


def test_zero_d2_takes_uniform_draw():
    P = np.full((4, 2), 5.0)
    c = seed.kmeanspp(P, 3, [0.9, 0.1, 0.6], 0)
    assert np.all(c == 5.0)                         # every draw lands on an equal point


def test_lloyd_one_iteration_hand():
    # 0, 1, 10, 11: seeds 0 (u0 = 0) and 11 (prefix 0, 1, 101, 222 vs 0.5 * 222 = 111);
    # one Lloyd step: {0, 1} -> 0.5, {10, 11} -> 10.5
    P = np.array([[0.0], [1.0], [10.0], [11.0]])
    c0 = seed.kmeanspp(P, 2, [0.0, 0.5], 0)
    assert np.array_equal(c0[:, 0], [0.0, 11.0])
    c1 = seed.kmeanspp(P, 2, [0.0, 0.5], 1)
    assert np.array_equal(c1[:, 0], [0.5, 10.5])


def test_K1_centre_is_the_mean():
    rng = np.random.default_rng(3)
    P = rng.normal(size=(101, 4))
    c = seed.kmeanspp(P, 1, [0.4], 3)
    assert np.allclose(c[0], P.mean(0), rtol=0, atol=1e-14)
    lab, _ = seed.label_nearest(P, c)
    assert np.all(lab == 0)


def test_separated_blobs_recovered():
    rng = np.random.default_rng(5)
    K, per = 5, 40
    true_c = rng.uniform(-1000, 1000, size=(K, 3))
    P = np.concatenate([true_c[c] + rng.normal(size=(per, 3)) for c in range(K)])
    truth = np.repeat(np.arange(K), per)
    c = seed.kmeanspp(P, K, rng.uniform(size=K), 5)
    lab, _ = seed.label_nearest(P, c)
    # the partition is the blob partition (up to a relabelling), the centres the blob means
    perm = {int(t): int(l) for t, l in zip(truth, lab)}
    assert len(set(perm.values())) == K
    assert np.all(lab == np.array([perm[int(t)] for t in truth]))
    for t in range(K):
        assert np.allclose(c[perm[t]], P[truth == t].mean(0), rtol=0, atol=1e-9)


def test_lloyd_fixed_point_brute_force():
    # converged Lloyd: every point's label is its nearest centre (brute-force norms), every centre
    # the mean of its points
    rng = np.random.default_rng(7)
    P = rng.normal(size=(300, 2))
    c = seed.kmeanspp(P, 4, rng.uniform(size=4), 100)
    dist = np.linalg.norm(P[:, None, :] - c[None, :, :], axis=2)
    lab = dist.argmin(1)
    assert np.array_equal(seed.nearest(P, c), lab)
    for e in range(4):
        assert np.allclose(c[e], P[lab == e].mean(0), rtol=0, atol=1e-12)


def test_nearest_ties_lowest_index():
    c = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]])
    assert seed.nearest(np.array([[0.0, 0.0]]), c)[0] == 0
    assert seed.nearest(np.array([[0.0, 0.0]]), c[::-1])[0] == 0
    assert seed.nearest(np.array([[-0.5, 0.5]]), c)[0] == 1


def test_empty_cluster_repair_hand():
    mu = np.array([[0.0], [1.0], [2.0], [10.0]])
    lab, c = seed.label_nearest(mu, np.array([[0.0], [100.0]]))
    assert np.array_equal(lab, [0, 0, 0, 1]) and c[1, 0] == 10.0
    # equal points: the lowest-index member of the only non-singleton cluster moves
    lab, c = seed.label_nearest(np.full((3, 1), 5.0), np.array([[5.0], [5.0]]))
    assert np.array_equal(lab, [1, 0, 0])
    # two empty clusters; the singleton cluster's member (the farthest from its centre) never moves
    mu = np.array([[0.0], [1.0], [3.0], [60.0]])
    lab, c = seed.label_nearest(mu, np.array([[0.0], [-100.0], [50.0], [-200.0]]))
    assert np.array_equal(lab, [0, 3, 1, 2]) and c[1, 0] == 3.0 and c[3, 0] == 1.0


def test_pick_members_hand():
    off = np.array([0, 3, 8, 10, 16, 17])            # m_k = 3, 5, 2, 6, 1
    labels = np.array([0, 0, 1, 0, 1])
    # cluster 0 with m = 3: big members 0, 1, 3 -> u = 0.5 -> position 1 -> member 1
    # cluster 1: no member with m_k >= 3 -> the largest (member 2, m_k = 2)
    assert np.array_equal(seed.pick_members(off, labels, 3, [0.5, 0.9]), [1, 2])
    assert np.array_equal(seed.pick_members(off, labels, 3, [0.99, 0.0]), [3, 2])
    assert np.array_equal(seed.pick_members(off, labels, 3, [0.0, 0.0, 0.3]), [0, 2, -1])
