"""Pins for the fp64 oracle (no GPU).  Each test checks the oracle against something other than
itself: hand-derived values, closed forms the paper fixes, invariants, metamorphic relations,
brute force on tiny inputs, or an independent library LP (scipy HiGHS).  The pin ids P1-P13
follow SURVEY.md §8(c); "P:n" = PAPER.md line n.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.optimize import linprog

import oracle
from paper_1510_00012_b200 import workloads as wl

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------------------- single formulas

def test_cost_hand_values():
    # c(x,y) = ||x-y||^2 (p=2): (0,0)-(3,4) -> 25; (1,2)-(3,4) -> 8
    C = oracle.cost([[0.0, 0.0], [1.0, 2.0]], [[3.0, 4.0], [1.0, 2.0]])
    np.testing.assert_array_equal(C, [[25.0, 5.0], [8.0, 0.0]])


def test_rho_golden():
    g = GOLD["rho_single_entry"]
    assert oracle.rho(g["x"], [0, 1], g["y"], g["rho0"]) == pytest.approx(g["rho"], rel=0, abs=1e-15)
    g = GOLD["rho_uniform_cost"]
    Y = np.array([p for mem in g["members"] for p in mem])
    off = np.cumsum([0] + [len(mem) for mem in g["members"]])
    assert oracle.rho(g["x"], off, Y, g["rho0"]) == pytest.approx(g["rho"], abs=1e-15)


def test_rho_is_rho0_times_mean_entry_cost():
    # reading X1: the mean is over all sum_k m*m_k plan entries (not divided again by N)
    x = np.array([[0.0], [10.0]])
    Y = np.array([[1.0], [2.0], [3.0]])            # member 0: {1,2}, member 1: {3}
    # costs by hand: row x=0: 1,4 | 9 ; row x=10: 81,64 | 49 ; sum = 208 over 6 entries
    assert oracle.rho(x, [0, 2, 3], Y, 2.0) == pytest.approx(2.0 * 208.0 / 6.0, abs=1e-12)


def test_pi1_2x2_hand():
    g = GOLD["pi1_2x2"]
    e = math.e
    om = np.array(g["omega"])
    want = np.array([[om[0] * e / (e + 1), om[1] / (e + 1)],
                     [om[0] / (e + 1), om[1] * e / (e + 1)]])
    P = oracle.pi1(np.full((2, 2), 0.25), np.zeros((2, 2)), g["C"], om, g["rho"], eps=0.0)
    np.testing.assert_allclose(P, want, rtol=1e-15, atol=0)
    P = oracle.pi1(np.full((2, 2), 0.25), np.zeros((2, 2)), g["C"], om, g["rho"], eps=1e-16)
    np.testing.assert_allclose(P, want, rtol=1e-14, atol=0)


def test_pi1_lambda_enters_like_cost():
    # Eq.badmmc0b: exp[(c+lambda)/(-rho)] -> lambda acts exactly like an added cost
    rng = np.random.default_rng(1)
    C, L = rng.random((3, 4)), rng.standard_normal((3, 4))
    P2, om = rng.random((3, 4)), rng.dirichlet(np.ones(4))
    a = oracle.pi1(P2, L, C, om, 0.7, 0.0)
    b = oracle.pi1(P2, np.zeros((3, 4)), C + L, om, 0.7, 0.0)
    np.testing.assert_allclose(a, b, rtol=1e-14)
    # a larger cost on one entry lowers that entry's share of its column
    C2 = C.copy(); C2[1, 2] += 1.0
    c = oracle.pi1(P2, L, C2, om, 0.7, 0.0)
    assert c[1, 2] < a[1, 2] and c[0, 2] > a[0, 2]


def test_pi1_eps_floor_semantics():
    # X3: eps is added after the exp-multiply.  With every exp underflowing to exactly 0, each
    # entry is eps and Eq.badmmc0 gives pi1_ij = w_j / m (not 0/0).
    om = np.array([0.2, 0.8])
    C = np.full((4, 2), 1e5)
    P = oracle.pi1(np.full((4, 2), 0.125), np.zeros((4, 2)), C, om, 1.0, eps=1e-16)
    np.testing.assert_allclose(P, np.tile(om / 4, (4, 1)), rtol=1e-15)
    with np.errstate(invalid="ignore"):
        Pn = oracle.pi1(np.full((4, 2), 0.125), np.zeros((4, 2)), C, om, 1.0, eps=0.0)
    assert np.isnan(Pn).all()


def test_pi1_eps_floor_nonuniform_pi2():
    """X3, Eq.badmmc0b: eps is added AFTER the product Pi2 * exp(...).  With a
    NON-uniform Pi2 and every exp of a column underflowing, every entry of that column is exactly
    eps and Eq.badmmc0 gives pi1_ij = w_j / m whatever Pi2 is; eps inside the product
    (Pi2 * (exp + eps)) would give w_j * Pi2_ij / sum_l Pi2_lj instead.  Column 1 does not
    underflow and keeps its closed form."""
    om = np.array([0.2, 0.8])
    P2 = np.array([[0.05, 0.10], [0.30, 0.20], [0.15, 0.05], [0.01, 0.14]])
    C = np.array([[1e5, 0.0], [1e5, 1.0], [1e5, 2.0], [1e5, 0.5]])
    P = oracle.pi1(P2, np.zeros((4, 2)), C, om, 1.0, eps=1e-16)
    np.testing.assert_allclose(P[:, 0], np.full(4, 0.2 / 4), rtol=1e-15)
    a = P2[:, 1] * np.exp(-C[:, 1]) + 1e-16
    np.testing.assert_allclose(P[:, 1], 0.8 * a / a.sum(), rtol=1e-14)
    # the same through Lambda: a huge dual on a column acts like a huge cost
    L = np.zeros((4, 2)); L[:, 0] = 1e5
    P = oracle.pi1(P2, L, np.zeros((4, 2)), om, 1.0, eps=1e-16)
    np.testing.assert_allclose(P[:, 0], np.full(4, 0.05), rtol=1e-15)


def test_pi1_tilde_eps_presence_and_placement():
    """X3, Eq.badmmc1b: pt1 = pi1 * exp(lambda / rho) + eps.  A row whose exps all
    underflow (lambda = -1e4 rho) is EXACTLY eps (not 0: eps dropped; not pi1 * eps: eps inside
    the product), and Eq.badmmc1 then spreads w_i evenly over the row: w_i / m_k."""
    rho = 0.37
    P1 = np.array([[0.2, 0.3, 0.05], [0.1, 0.4, 0.25]])
    L = np.array([[-1e4 * rho] * 3, [0.0, rho * math.log(2.0), -rho * math.log(4.0)]])
    B = oracle.pi1_tilde(P1, L, rho, eps=1e-16)
    np.testing.assert_array_equal(B[0], np.full(3, 1e-16))
    np.testing.assert_allclose(B[1], [0.1 + 1e-16, 0.8 + 1e-16, 0.0625 + 1e-16], rtol=1e-15)
    w = np.array([0.3, 0.7])
    P2 = oracle.pi2(B, w)
    np.testing.assert_allclose(P2[0], np.full(3, 0.1), rtol=1e-15)                 # w_0 / m_k
    np.testing.assert_allclose(P2[1], 0.7 * np.array([0.1, 0.8, 0.0625]) / 0.9625, rtol=1e-14)
    # eps = 0: the underflowed row has no mass and Eq.badmmc1 is 0/0
    with np.errstate(invalid="ignore"):
        assert np.isnan(oracle.pi2(oracle.pi1_tilde(P1, L, rho, eps=0.0), w)[0]).all()


def test_pi1_single_row_and_zero_cost():
    om = np.array([0.1, 0.6, 0.3])
    P = oracle.pi1(np.array([[0.2, 0.5, 0.3]]), np.ones((1, 3)), np.ones((1, 3)) * 3, om, 1.0)
    np.testing.assert_allclose(P, om[None], rtol=1e-15)              # m=1: forced
    P2 = np.array([[0.1, 0.2], [0.3, 0.4]])
    P = oracle.pi1(P2, np.zeros((2, 2)), np.zeros((2, 2)), np.array([0.5, 0.5]), 1.0, eps=0.0)
    np.testing.assert_allclose(P, [[0.5 * 0.1 / 0.4, 0.5 * 0.2 / 0.6], [0.5 * 0.3 / 0.4, 0.5 * 0.4 / 0.6]],
                               rtol=1e-15)


def test_pi1_tilde_hand():
    # lambda=[[rho ln2, 0],[0,0]] doubles entry (1,1)
    rho = 0.37
    P1 = np.array([[0.1, 0.2], [0.3, 0.4]])
    L = np.array([[rho * math.log(2.0), 0.0], [0.0, 0.0]])
    B = oracle.pi1_tilde(P1, L, rho, eps=1e-16)
    np.testing.assert_allclose(B, [[0.2 + 1e-16, 0.2 + 1e-16], [0.3 + 1e-16, 0.4 + 1e-16]], rtol=1e-15)


def test_pi2_hand():
    B = np.array([[1.0, 3.0], [2.0, 2.0]])
    w = np.array([0.4, 0.6])
    np.testing.assert_allclose(oracle.pi2(B, w), [[0.1, 0.3], [0.3, 0.3]], rtol=1e-15)
    np.testing.assert_allclose(oracle.pi2(np.array([[5.0], [7.0]]), w), [[0.4], [0.6]], rtol=1e-15)  # m_k=1


def test_rowmass_hand():
    r, wt = oracle.rowmass(np.array([[1.0, 3.0], [2.0, 2.0], [0.0, 2.0]]))
    np.testing.assert_allclose(r, [4.0, 4.0, 2.0]); np.testing.assert_allclose(wt, [0.4, 0.4, 0.2])


def test_consensus_golden():
    for case in GOLD["consensus"]["cases"]:
        np.testing.assert_allclose(oracle.consensus(case["wt"], 0), case["R1"], rtol=1e-15)
        np.testing.assert_allclose(oracle.consensus(case["wt"], 1), case["R2"], rtol=1e-7)
    v = np.array([[0.2, 0.5, 0.3]])
    for rule in (0, 1):
        np.testing.assert_allclose(oracle.consensus(v, rule), v[0], rtol=1e-15)     # N=1
        np.testing.assert_allclose(oracle.consensus(np.repeat(v, 5, 0), rule), v[0], rtol=1e-14)


def test_dual_hand():
    L = np.array([[1.0, -2.0]])
    np.testing.assert_array_equal(oracle.dual(L, [[0.3, 0.7]], [[0.3, 0.7]], 5.0), L)
    np.testing.assert_allclose(oracle.dual(L, [[1.5, 1.0]], [[0.5, 0.0]], 1.0), [[2.0, -1.0]])


def test_update_support_golden():
    g = GOLD["update_support_2members"]
    x = oracle.update_support(np.zeros((2, 1)), [0.5, 0.5], [0, 2, 3], np.array([[0.0], [2.0], [4.0]]),
                              [np.array([[0.4, 0.1], [0.2, 0.3]]), np.array([[0.5], [0.5]])])
    np.testing.assert_allclose(x, g["x_expected"], rtol=1e-15)
    # X12: w_i < 1e-12 keeps x_i
    x = oracle.update_support(np.array([[7.0], [9.0]]), [1.0, 0.0], [0, 1], np.array([[1.0]]),
                              [np.array([[1.0], [0.0]])])
    np.testing.assert_array_equal(x, [[1.0], [9.0]])


# ----------------------------------------------------------------------------- Alg. 4 end to end

def _cluster(N=12, m=4, d=2, seed=3, mk=(1, 6), alpha=1.0, spread=1.0):
    b = wl.make_random(N, m, d, K=1, mk_range=mk, seed=seed, dtype="f64", alpha=alpha, spread=spread)
    return b


def _run(b, T, tau, rule=0, eps=1e-16, **kw):
    return oracle.badmm_centroid(b.x0[0], b.w0[0], b.offsets, b.supports, b.weights, T, tau, rule,
                                 2.0, eps, **kw)


@pytest.mark.parametrize("rule", [0, 1])
def test_P1_P2_P3_marginals_simplex_dual_sum(rule):
    b = _cluster(N=20, m=5, d=3, seed=5)
    res = _run(b, T=23, tau=7, rule=rule)
    assert abs(res.w.sum() - 1) < 1e-12 and (res.w >= 0).all()                      # P2
    for k in range(b.N):
        _, om = b.member(k)
        P1, P2, L = res.member("Pi1", k), res.member("Pi2", k), res.member("Lam", k)
        np.testing.assert_allclose(P1.sum(0), om / om.sum(), rtol=1e-12)             # P1: columns
        np.testing.assert_allclose(P2.sum(1), res.w, rtol=1e-12)                     # P1: rows
        assert (P1 > 0).all() and (P2 > 0).all()
        assert abs(L.sum()) <= 1e-12 * res.rho                                        # P3


def test_alg4_one_iteration_hand_values():
    """ONE iteration of Alg. 4 from the product init, every quantity by hand (two members, N = 2,
    so that the consensus w differs from each member's row mass and Pi2 != Pi1).
    x = (0, 1) on a line; both members have y = (0, 1), omega^A = (.3, .7), omega^B = (.6, .4);
    w0 = (.5, .5).  C = [[0,1],[1,0]] for both, mean entry cost 1/2, so rho = 2 x 1/2 = 1 (X1;
    the literal Eq.rho's extra 1/N would give 1/2).  Eq.badmmc0b/c0 with Pi2^0 = w0 (x) omega:
    Pi1_ij = omega_j e^{-C_ij} / (1 + e^-1) (the w0 and omega factors cancel per column).
    Lambda^0 = 0, so pt1 = Pi1 + eps, r^k_i = row sums, w = (r^A + r^B)/2 (R1, N = 2, the r's are
    already normalised), Pi2_ij = Pi1_ij w_i / r_i (Eq.badmmc1), Lambda = rho (Pi1 - Pi2)
    (Eq.badmm2), and the surrogate objective (X14) is
    (1/N) sum_k <C, Pi1^k> = (1/2)((.7 + .3) + (.4 + .6)) / (e + 1) = 1 / (e + 1)."""
    e = math.e
    Y = np.array([[0.0], [1.0], [0.0], [1.0]])
    om = np.array([0.3, 0.7, 0.6, 0.4])
    res = oracle.badmm_centroid([[0.0], [1.0]], [0.5, 0.5], [0, 2, 4], Y, om, 1, 10 ** 6, 0, 2.0, 1e-16)
    assert res.rho == pytest.approx(1.0, rel=1e-15)
    P1 = {}
    r = {}
    for k, (a, b) in enumerate(((0.3, 0.7), (0.6, 0.4))):
        P1[k] = np.array([[a * e, b], [a, b * e]]) / (e + 1)
        r[k] = P1[k].sum(1)
        np.testing.assert_allclose(res.member("Pi1", k), P1[k], rtol=1e-14)
    w = (r[0] + r[1]) / 2
    np.testing.assert_allclose(res.w, w, rtol=1e-14)
    for k in range(2):
        P2 = P1[k] * (w / r[k])[:, None]
        np.testing.assert_allclose(res.member("Pi2", k), P2, rtol=1e-14)
        np.testing.assert_allclose(res.member("Lam", k), 1.0 * (P1[k] - P2), rtol=1e-12, atol=1e-16)
    assert res.obj == pytest.approx(1.0 / (e + 1.0), rel=1e-14)
    # a cheaper entry count check of X1 inside Alg. 4 (N = 2, unequal m_k): T = 0 returns rho only
    r0 = oracle.badmm_centroid([[0.0], [10.0]], [0.5, 0.5], [0, 2, 3], [[1.0], [2.0], [3.0]], [0.4, 0.6, 1.0], 0, 1)
    assert r0.rho == pytest.approx(2.0 * 208.0 / 6.0, rel=1e-15)


def test_alg4_init_product_and_warm_hand_values():
    """Alg. 4's initialisation (P:686 with P:842-850): a cold member starts from the product
    Pi2^0_ij = w0_i omega_j, a warm member from its given Pi2.  Same geometry as above (C =
    [[0,1],[1,0]], rho = 1) with a NON-uniform w0 = (.4, .6); member A warm from
    Pi2^w = [[.1, .2], [.25, .45]], member B cold.  After one iteration, by Eq.badmmc0b/c0:
    Pi1_ij = P_ij e^{-C_ij} omega_j / sum_l P_lj e^{-C_lj} with P = Pi2^w (A) or w0 (x) omega (B)."""
    e1 = math.exp(-1.0)
    Y = np.array([[0.0], [1.0], [0.0], [1.0]])
    om = np.array([0.3, 0.7, 0.6, 0.4])
    Pw = np.array([[0.1, 0.2], [0.25, 0.45]])
    w0 = np.array([0.4, 0.6])
    res = oracle.badmm_centroid([[0.0], [1.0]], w0, [0, 2, 4], Y, om, 1, 10 ** 6, 0, 2.0, 1e-16,
                                warm=[Pw, np.zeros((2, 2))], warm_mask=[1, 0])
    G = np.array([[1.0, e1], [e1, 1.0]])
    for k, P in ((0, Pw * G), (1, np.outer(w0, om[2:]) * G)):
        want = P / P.sum(0) * om[2 * k:2 * k + 2]
        np.testing.assert_allclose(res.member("Pi1", k), want, rtol=1e-13)


@pytest.mark.parametrize("T,tau", [(3, 3), (6, 3)])
def test_support_update_is_eq_updatex_on_pi2(T, tau):
    """X5 / Eq.updatex: x_i = 1/(N w_i) sum_k sum_j pi_ij^(k) x_j^(k) holds LITERALLY
    (with the paper's 1/(N w_i), not the oracle's measured row mass) for the coupling whose rows
    sum to w_i, i.e. Pi^(2) (Eq.badmmc1).  Right after the support update at t = T (a multiple of
    tau) the returned Pi2, w and x are the ones the update used."""
    b = _cluster(N=7, m=4, d=3, seed=29, mk=(2, 6))
    res = _run(b, T=T, tau=tau)
    num = np.zeros((b.m, b.d))
    for k in range(b.N):
        y, _ = b.member(k)
        num += res.member("Pi2", k) @ y
    np.testing.assert_allclose(res.x, num / (b.N * res.w[:, None]), rtol=1e-12, atol=1e-13)
    # and not for Pi1: its rows do not sum to w_i (the identity would fail visibly)
    num1 = sum(res.member("Pi1", k) @ b.member(k)[0] for k in range(b.N))
    assert np.abs(num1 / (b.N * res.w[:, None]) - res.x).max() > 1e-6


@pytest.mark.parametrize("n_iter", [1, 5, 25])
def test_P4_gibbs_form_of_pi2(n_iter):
    """With eps = 0 and fixed support, Lambda cancels out of the Pi^(2) recursion
    (Eq.badmmc0b * Eq.badmmc1b) so Pi^(2),n = diag(u) exp(-n C/rho) diag(v) from the product
    init (derived from P:590-602).  Double differences of log Pi2 + nC/rho must vanish."""
    b = _cluster(N=6, m=4, d=2, seed=11)
    res = _run(b, T=n_iter, tau=10 ** 6, eps=0.0)
    for k in range(b.N):
        y, _ = b.member(k)
        C = ((b.x0[0][:, None, :] - y[None, :, :]) ** 2).sum(-1)
        G = np.log(res.member("Pi2", k)) + n_iter * C / res.rho
        D = G - G[:, :1] - G[:1, :] + G[0, 0]
        assert np.abs(D).max() < 1e-9 * max(1.0, np.abs(G).max())
    # and Lambda itself is far from separable (it is not what cancels trivially)
    L = res.member("Lam", 0)
    if n_iter > 1 and L.shape[1] > 1:
        DL = L - L[:, :1] - L[:1, :] + L[0, 0]
        assert np.abs(DL).max() > 1e-6 * res.rho


@pytest.mark.parametrize("rule", [0, 1])
def test_P5_single_support_point(rule):
    """m = 1 reduces to K-means on distribution means."""
    b = _cluster(N=9, m=1, d=3, seed=2)
    res = _run(b, T=10, tau=5, rule=rule)
    assert res.w[0] == 1.0
    xs = np.zeros(3)
    for k in range(b.N):
        y, om = b.member(k)
        np.testing.assert_allclose(res.member("Pi1", k)[0], om, rtol=1e-14)
        np.testing.assert_allclose(res.member("Pi2", k)[0], om, rtol=1e-14, atol=1e-15)
        assert np.abs(res.member("Lam", k)).max() < 1e-13 * res.rho
        xs += om @ y
    np.testing.assert_allclose(res.x[0], xs / b.N, rtol=1e-13)
    obj = np.mean([om @ ((y - res.x[0]) ** 2).sum(1) for y, om in (b.member(k) for k in range(b.N))])
    assert res.obj == pytest.approx(obj, rel=1e-13)


@pytest.mark.parametrize("rule", [0, 1])
def test_P6_single_member_is_its_own_barycenter(rule):
    """N = 1 and init = the member -> the member is the barycenter (objective 0).  Points well
    separated relative to rho (= 2 x mean cost): close points can settle in a shared local
    stationary point, since Alg. 4 is a heuristic."""
    y = np.array([[0.0, 0.0], [3.0, 0.0], [0.0, 3.0], [3.0, 3.0], [1.5, 6.0]])
    om = np.array([0.1, 0.3, 0.2, 0.25, 0.15])
    res = oracle.badmm_centroid(y, np.full(5, 0.2), [0, 5], y, om, 100, 10, rule)
    np.testing.assert_allclose(res.w, om, atol=1e-5)
    np.testing.assert_allclose(res.x, y, atol=1e-5)
    assert res.obj < 1e-5
    assert oracle.exact_objective(res.x, res.w, [0, 5], y, om) < 1e-5


def test_P7_two_point_masses():
    g = GOLD["two_point_masses"]
    Y = np.array(g["members"])
    res = oracle.badmm_centroid([[0.3]], [1.0], [0, 1, 2], Y, [1.0, 1.0], 10, 1, 0)
    assert res.x[0, 0] == pytest.approx(g["x"], abs=1e-12)
    assert res.obj == pytest.approx(g["objective"], abs=1e-12)
    assert oracle.exact_objective(res.x, res.w, [0, 1, 2], Y, [1.0, 1.0]) == pytest.approx(1.0, abs=1e-12)


def _fullbatch_lp(x, offsets, Y, omega):
    """Eq.fullbatch-lp at fixed x: min_{Pi, w} sum_k <C_k, Pi_k>, rows = w, cols = w^(k)."""
    m = x.shape[0]
    N = len(offsets) - 1
    sizes = np.diff(offsets)
    nv = m * int(sizes.sum()) + m
    c = np.zeros(nv)
    A, rhs = [], []
    base = 0
    for k in range(N):
        y = Y[offsets[k]:offsets[k + 1]]
        om = omega[offsets[k]:offsets[k + 1]]
        mk = sizes[k]
        c[base:base + m * mk] = ((x[:, None, :] - y[None]) ** 2).sum(-1).ravel()
        for i in range(m):                                   # sum_j pi_ij - w_i = 0
            row = np.zeros(nv); row[base + i * mk: base + (i + 1) * mk] = 1; row[nv - m + i] = -1
            A.append(row); rhs.append(0.0)
        for j in range(mk):                                  # sum_i pi_ij = w_j^(k)
            row = np.zeros(nv); row[base + j: base + m * mk: mk] = 1
            A.append(row); rhs.append(om[j] / om.sum())
        base += m * mk
    row = np.zeros(nv); row[nv - m:] = 1; A.append(row); rhs.append(1.0)
    r = linprog(c, A_eq=np.array(A), b_eq=np.array(rhs), bounds=(0, None), method="highs")
    assert r.status == 0
    return r.fun / N


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_P8_lp_lower_bound(seed):
    b = _cluster(N=4, m=3, d=2, seed=20 + seed, mk=(2, 4))
    res = _run(b, T=2000, tau=10 ** 6)                       # fixed support
    lp = _fullbatch_lp(b.x0[0], b.offsets, b.supports, b.weights)
    exact = oracle.exact_objective(b.x0[0], res.w, b.offsets, b.supports, b.weights)
    assert exact >= lp - 1e-9                                 # hard: LP is the optimum over w
    assert exact <= lp * 1.10 + 1e-12                         # soft: B-ADMM is near it


def test_P10_metamorphic_scale_translate_permute():
    b = _cluster(N=10, m=4, d=2, seed=13)
    base = _run(b, T=20, tau=5)
    s, t = 3.7, np.array([2.0, -1.5])
    bs = wl.replace(b, supports=b.supports * s + t, x0=b.x0 * s + t)
    r2 = _run(bs, T=20, tau=5)
    np.testing.assert_allclose(r2.w, base.w, rtol=1e-10)
    np.testing.assert_allclose(r2.x, base.x * s + t, rtol=1e-10, atol=1e-10)
    assert r2.obj == pytest.approx(base.obj * s * s, rel=1e-10)
    assert r2.rho == pytest.approx(base.rho * s * s, rel=1e-12)
    perm = np.random.default_rng(0).permutation(b.N)
    bp = b.subset(perm)
    r3 = _run(bp, T=20, tau=5)
    np.testing.assert_allclose(r3.w, base.w, rtol=1e-12)
    np.testing.assert_allclose(r3.x, base.x, rtol=1e-12)
    for kk, k in enumerate(perm):
        np.testing.assert_allclose(r3.member("Pi1", kk), base.member("Pi1", k), rtol=1e-10, atol=1e-18)


def test_P10_column_permutation():
    b = _cluster(N=3, m=3, d=2, seed=17, mk=(4, 4))
    base = _run(b, T=7, tau=3)
    perm = np.array([2, 0, 3, 1])
    idx = np.concatenate([b.offsets[k] + perm for k in range(b.N)])
    bp = wl.replace(b, supports=b.supports[idx], weights=b.weights[idx])
    r = _run(bp, T=7, tau=3)
    for k in range(b.N):
        np.testing.assert_allclose(r.member("Pi1", k), base.member("Pi1", k)[:, perm], rtol=1e-11)


def test_P11_support_in_convex_hull():
    b = _cluster(N=8, m=3, d=2, seed=19)
    res = _run(b, T=10, tau=5)
    Y = b.supports
    for i in range(3):
        r = linprog(np.zeros(len(Y)), A_eq=np.vstack([Y.T, np.ones(len(Y))]),
                    b_eq=np.concatenate([res.x[i], [1.0]]), bounds=(0, None), method="highs")
        assert r.status == 0


# ----------------------------------------------------------------------------- exact OT

def _brute_force_ot(a, b, c):
    """Minimum over all basic feasible solutions of the transport polytope (vertex enumeration)."""
    ma, mb = c.shape
    cells = list(itertools.product(range(ma), range(mb)))
    A = np.zeros((ma + mb, ma * mb))
    for i, j in cells:
        A[i, i * mb + j] = 1
        A[ma + j, i * mb + j] = 1
    rhs = np.concatenate([a, b])
    best = np.inf
    for S in itertools.combinations(range(ma * mb), ma + mb - 1):
        As = A[:, S]
        if np.linalg.matrix_rank(As) < ma + mb - 1:
            continue
        sol, *_ = np.linalg.lstsq(As, rhs, rcond=None)
        if (sol < -1e-12).any() or np.abs(As @ sol - rhs).max() > 1e-10:
            continue
        best = min(best, float(c.ravel()[list(S)] @ sol))
    return best


@pytest.mark.parametrize("seed", range(6))
def test_P12_transport_vs_vertex_enumeration(seed):
    rng = np.random.default_rng(seed)
    ma, mb = rng.integers(1, 4, size=2)
    a, b = rng.dirichlet(np.ones(ma)), rng.dirichlet(np.ones(mb))
    c = rng.random((ma, mb)) * 5
    assert oracle.transport(a, b, c) == pytest.approx(_brute_force_ot(a, b, c), abs=1e-9)


@pytest.mark.parametrize("seed", range(5))
def test_P12_transport_vs_linprog(seed):
    rng = np.random.default_rng(100 + seed)
    ma, mb = rng.integers(3, 12, size=2)
    a, b = rng.dirichlet(np.ones(ma) * 0.5), rng.dirichlet(np.ones(mb))
    c = rng.random((ma, mb))
    if seed == 0:
        c = np.round(c * 3)                                        # ties / degeneracy
    A = np.zeros((ma + mb, ma * mb))
    for i in range(ma):
        A[i, i * mb:(i + 1) * mb] = 1
    for j in range(mb):
        A[ma + j, j::mb] = 1
    r = linprog(c.ravel(), A_eq=A, b_eq=np.concatenate([a, b]), bounds=(0, None), method="highs")
    W, plan = oracle.transport(a, b, c, want_plan=True)
    assert W == pytest.approx(r.fun, abs=1e-10)
    np.testing.assert_allclose(plan.sum(1), a, atol=1e-12)
    np.testing.assert_allclose(plan.sum(0), b, atol=1e-12)
    assert (plan >= 0).all()


def test_P12_transport_identities_and_1d_monotone():
    rng = np.random.default_rng(5)
    x, w = rng.standard_normal((5, 2)), rng.dirichlet(np.ones(5))
    y, v = rng.standard_normal((4, 2)), rng.dirichlet(np.ones(4))
    assert oracle.w2sq(x, w, x, w) == pytest.approx(0.0, abs=1e-14)
    assert oracle.w2sq(x, w, y, v) == pytest.approx(oracle.w2sq(y, v, x, w), abs=1e-12)
    # 1-D: W2^2 = int_0^1 |F^-1(t) - G^-1(t)|^2 dt (quantile coupling)
    xa, xb = np.sort(rng.standard_normal(6)), np.sort(rng.standard_normal(7))
    wa, wb = rng.dirichlet(np.ones(6)), rng.dirichlet(np.ones(7))
    Fa, Fb = np.cumsum(wa), np.cumsum(wb)
    ts = np.unique(np.concatenate([[0.0], Fa[:-1], Fb[:-1], [1.0]]))
    q = 0.0
    for t0, t1 in zip(ts[:-1], ts[1:]):
        tm = 0.5 * (t0 + t1)
        q += (t1 - t0) * (xa[np.searchsorted(Fa, tm)] - xb[np.searchsorted(Fb, tm)]) ** 2
    assert oracle.w2sq(xa[:, None], wa, xb[:, None], wb) == pytest.approx(q, abs=1e-12)


def test_P13_1d_barycenter_vs_quantile_average():
    """1-D free-support barycenter: the quantile-average distribution is the exact barycenter,
    so B-ADMM's exact objective cannot be below it (soft: within a few %)."""
    rng = np.random.default_rng(9)
    N, mk = 6, 5
    Y = rng.standard_normal((N * mk, 1))
    om = np.tile(np.full(mk, 1.0 / mk), N)
    off = np.arange(N + 1) * mk
    # exact barycenter of uniform 5-point measures: sorted points averaged rank by rank
    sortedY = np.sort(Y.reshape(N, mk), axis=1)
    bx = sortedY.mean(0)
    opt = np.mean([oracle.w2sq(bx[:, None], om[:mk], sortedY[k][:, None], om[:mk]) for k in range(N)])
    res = oracle.badmm_centroid(Y[:mk], np.full(mk, 1.0 / mk), off, Y, om, 200, 10, 0)
    ex = oracle.exact_objective(res.x, res.w, off, Y, om)
    assert ex >= opt - 1e-10
    assert ex <= opt * 1.2 + 1e-12


def test_oracle_thread_count_does_not_change_results():
    b = _cluster(N=40, m=4, d=2, seed=23)
    r1 = _run(b, T=12, tau=4, nthreads=1)
    r4 = _run(b, T=12, tau=4, nthreads=4)
    np.testing.assert_array_equal(r1.Pi1, r4.Pi1)
    np.testing.assert_array_equal(r1.x, r4.x)
    np.testing.assert_array_equal(r1.w, r4.w)


def test_oracle_errors():
    with pytest.raises(oracle.OracleError, match="zero_rho"):
        oracle.badmm_centroid([[1.0]], [1.0], [0, 1], [[1.0]], [1.0], 5, 5)
    with pytest.raises(oracle.OracleError, match="arg"):
        oracle.badmm_centroid([[1.0]], [1.0], [0, 2], [[1.0], [2.0]], [0.5, 0.4], 5, 5)


# ---------------------------------------------------------------- O7 assignment (Alg. 1)

def _w2_1d(xa, wa, xb, wb):
    """1-D W2^2 by the quantile coupling (closed form, independent of the transport simplex)."""
    ia, ib = np.argsort(xa), np.argsort(xb)
    xa, wa, xb, wb = xa[ia], wa[ia] / wa.sum(), xb[ib], wb[ib] / wb.sum()
    Fa, Fb = np.cumsum(wa), np.cumsum(wb)
    ts = np.unique(np.concatenate([[0.0], Fa[:-1], Fb[:-1], [1.0]]))
    q = 0.0
    for t0, t1 in zip(ts[:-1], ts[1:]):
        tm = 0.5 * (t0 + t1)
        q += (t1 - t0) * (xa[min(np.searchsorted(Fa, tm), len(xa) - 1)] - xb[min(np.searchsorted(Fb, tm), len(xb) - 1)]) ** 2
    return q


def test_O7_assign_1d_closed_form():
    """Labels / best / second-best W^2 against the 1-D quantile formula for every (member, centroid)."""
    rng = np.random.default_rng(11)
    K, m, N = 5, 4, 40
    x = rng.normal(0, 3, (K, m, 1))
    w = rng.dirichlet(np.ones(m), K) * 1.7                       # unnormalised: renormalised inside
    sizes = rng.integers(1, 7, N)
    off = np.concatenate([[0], np.cumsum(sizes)])
    Y = rng.normal(0, 3, (off[-1], 1))
    om = rng.dirichlet(np.ones(off[-1]))                          # per member renormalised inside
    lab, best, second = oracle.assign(x, w, off, Y, om)
    for k in range(N):
        a, b = off[k], off[k + 1]
        W = np.array([_w2_1d(x[c, :, 0], w[c], Y[a:b, 0], om[a:b]) for c in range(K)])
        order = np.argsort(W, kind="stable")
        assert lab[k] == order[0]
        assert best[k] == pytest.approx(W[order[0]], abs=1e-10)
        assert second[k] == pytest.approx(W[order[1]], abs=1e-10)


def test_O7_assign_identity_and_ties():
    """A member equal to centroid c is assigned to c with W^2 = 0; duplicated centroids tie and the
    lowest index wins (X13); translating everything leaves the labels unchanged."""
    rng = np.random.default_rng(12)
    K, m, d = 4, 3, 2
    x = rng.normal(0, 5, (K, m, d))
    x[3] = x[1]                                                   # centroid 3 duplicates centroid 1
    w = rng.dirichlet(np.ones(m), K)
    w[3] = w[1]
    off = np.arange(K + 1) * m
    Y = x.reshape(-1, d).copy()
    om = w.reshape(-1).copy()
    lab, best, second = oracle.assign(x, w, off, Y, om)
    assert list(lab) == [0, 1, 2, 1]
    assert np.abs(best).max() < 1e-12
    assert second[1] < 1e-12 and second[3] < 1e-12 and second[0] > 1e-3
    lab2, best2, _ = oracle.assign(x + 7.5, w, off, Y + 7.5, om)
    assert list(lab2) == list(lab) and np.abs(best2).max() < 1e-10


def test_O8_outer_loop_recovers_separated_groups():
    """Two groups of distributions 40 units apart, initial labels with 1/4 of each group swapped:
    round 1's centroids are barycenters of 3:1 mixtures and lie on their majority's side, so the
    exact assignment recovers the groups (changed fraction = 1/4), round 2 changes nothing and
    the loop stops (the label-change rule with stop_frac = 0)."""
    from paper_1510_00012_b200 import workloads as wl
    rng = np.random.default_rng(21)
    N, m, d = 40, 3, 2
    truth = np.repeat([0, 1], N // 2).astype(np.int32)
    sizes = rng.integers(2, 6, N)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    centre = np.where(truth[:, None] == 0, -20.0, 20.0)
    Y = np.repeat(centre, sizes, axis=0) + rng.normal(0, 1, (off[-1], d))
    W = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
    lab0 = truth.copy()
    flip = np.concatenate([rng.choice(N // 2, N // 8, replace=False), N // 2 + rng.choice(N // 2, N // 8, replace=False)])
    lab0[flip] = 1 - lab0[flip]
    x0 = np.stack([Y[off[k]:off[k] + m] if sizes[k] >= m else np.resize(Y[off[k]:off[k + 1]], (m, d))
                   for k in (0, N - 1)])
    w0 = np.full((2, m), 1.0 / m)
    b = wl.Bundle("two_groups", d, m, 2, off, Y, W, lab0, x0, w0, "f64", wl.Schedule(T=20, tau=10))
    lab, rounds, changed, objs, x, w = oracle.cluster(b, 20, 10, 5)
    np.testing.assert_array_equal(lab, truth)
    assert rounds == 2 and changed[0] == pytest.approx(0.25) and changed[1] == 0.0
    assert (x[0] < 0).all() and (x[1] > 0).all()


# ---------------------------------------------------------------- symbolic supports

def test_symbolic_table_equals_euclidean_with_fixed_support():
    """With D[a, b] = |e_a - e_b|^2 for an embedding e of the symbols, the symbolic mode is the
    Euclidean mode on the embedded points with the support update skipped: run both for T < tau
    (Euclidean never updates x before tau iterations, X6) and compare plans, w and objective."""
    rng = np.random.default_rng(31)
    V, m, N = 40, 5, 12
    emb = rng.normal(0, 1, (V, 3))
    D = ((emb[:, None, :] - emb[None, :, :]) ** 2).sum(-1)
    xs = rng.choice(V, m, replace=False)
    sizes = rng.integers(1, 8, N)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ys = rng.integers(0, V, off[-1])
    om = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
    w0 = rng.dirichlet(np.ones(m))
    T = 7
    a = oracle.badmm_table(xs, w0, off, ys, om, D, T)
    b = oracle.badmm_centroid(emb[xs], w0, off, emb[ys], om, T, T + 1)
    assert a.rho == pytest.approx(b.rho, rel=1e-13)
    np.testing.assert_allclose(a.w, b.w, rtol=1e-12, atol=1e-15)
    assert a.obj == pytest.approx(b.obj, rel=1e-12)
    for k in range(N):
        np.testing.assert_allclose(a.mats["Pi1"][k], b.mats["Pi1"][k], rtol=1e-11, atol=1e-16)


def test_symbolic_table_orientation_hand():
    """Symbolic supports: C^(k)_ij = D[centroid symbol x_i][member symbol y_j].  A
    NON-symmetric table tells the orientation apart.  m = 1 forces Pi1 = omega, so the
    surrogate objective is sum_j omega_j D[x_0][y_j] and rho = 2 x mean_j D[x_0][y_j]."""
    D = np.array([[0.0, 1.0, 4.0], [2.0, 0.0, 5.0], [7.0, 3.0, 0.0]])
    res = oracle.badmm_table([0], [1.0], [0, 2], [1, 2], [0.25, 0.75], D, 3)
    assert res.rho == pytest.approx(2.0 * (1.0 + 4.0) / 2, rel=1e-15)               # transposed: 9
    assert res.obj == pytest.approx(0.25 * 1.0 + 0.75 * 4.0, rel=1e-15)              # transposed: 5.75
    np.testing.assert_allclose(res.mats["Pi1"][0], [[0.25, 0.75]], rtol=1e-15)
    # m = 2, one member with one point: C = (D[0][1], D[2][1]) = (1, 3), rho = 2 x 2
    res = oracle.badmm_table([0, 2], [0.5, 0.5], [0, 1], [1], [1.0], D, 0)
    assert res.rho == pytest.approx(4.0, rel=1e-15)                                  # transposed: 7
    # N = 2 (X1 inside the symbolic mode): members {1} and {0, 2}: costs 1, 3 | 0, 4, 7, 0 -> 15 / 6
    res = oracle.badmm_table([0, 2], [0.5, 0.5], [0, 1, 3], [1, 0, 2], [1.0, 0.5, 0.5], D, 0)
    assert res.rho == pytest.approx(2.0 * 15.0 / 6.0, rel=1e-15)                     # 1/N typo: 2.5


def test_symbolic_support_is_never_updated_and_marginals_hold():
    rng = np.random.default_rng(32)
    V, m, N = 30, 4, 10
    D = rng.uniform(0.1, 3.0, (V, V))                         # any nonnegative table (not a metric)
    xs = rng.choice(V, m, replace=False)
    sizes = rng.integers(1, 6, N)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ys = rng.integers(0, V, off[-1])
    om = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
    res = oracle.badmm_table(xs, np.full(m, 1.0 / m), off, ys, om, D, 60)
    np.testing.assert_array_equal(res.x, xs)
    assert abs(res.w.sum() - 1) < 1e-12 and (res.w >= 0).all()
    for k in range(N):
        np.testing.assert_allclose(res.mats["Pi1"][k].sum(0), om[off[k]:off[k + 1]], rtol=1e-12)  # P1 columns
        np.testing.assert_allclose(res.mats["Pi2"][k].sum(1), res.w, rtol=1e-10, atol=1e-15)     # P1 rows


# ---------------------------------------------------------------- Eq.merge initialisation

def test_merge_init_pins():
    """Eq.merge: each step merges the pair minimising w_i w_j |x_i-x_j|^2/(w_i+w_j) (brute force
    over the pairs in the test) into the weighted mean; mass and mean are preserved; one merge
    moves the distribution by W^2(P, P') <= w_i|x_i - xb|^2 + w_j|x_j - xb|^2, which for
    the merged pair equals the merge cost; m >= m_k leaves the points (fallback splits)."""
    rng = np.random.default_rng(41)
    y = rng.normal(0, 2, (7, 3))
    w = rng.dirichlet(np.ones(7))
    # one merge, by brute force
    best, bi, bj = np.inf, -1, -1
    for i in range(7):
        for j in range(i + 1, 7):
            c = w[i] * w[j] * ((y[i] - y[j]) ** 2).sum() / (w[i] + w[j])
            if c < best:
                best, bi, bj = c, i, j
    x6, w6 = oracle.merge(y, w, 6)
    xb = (w[bi] * y[bi] + w[bj] * y[bj]) / (w[bi] + w[bj])
    keep = [k for k in range(7) if k not in (bi, bj)]
    np.testing.assert_allclose(x6[bi], xb, rtol=1e-14)
    assert w6[bi] == pytest.approx(w[bi] + w[bj], rel=1e-14)
    others = [k for k in range(6) if k != bi]
    np.testing.assert_allclose(x6[others], y[keep], rtol=0, atol=0)
    W = oracle.w2sq(y, w, x6, w6)
    bound = w[bi] * ((y[bi] - xb) ** 2).sum() + w[bj] * ((y[bj] - xb) ** 2).sum()
    assert W <= bound + 1e-12 and bound == pytest.approx(best, rel=1e-12)
    # full reduction: mass and mean preserved
    x3, w3 = oracle.merge(y, w, 3)
    assert w3.sum() == pytest.approx(1.0, abs=1e-15)
    np.testing.assert_allclose(w3 @ x3, w @ y, rtol=1e-12, atol=1e-12)
    # m >= m_k: the member itself (m = m_k) and heaviest-point splitting (m > m_k)
    x7, w7 = oracle.merge(y, w, 7)
    np.testing.assert_allclose(x7, y, atol=0)
    x9, w9 = oracle.merge(y, w, 9)
    h = int(np.argmax(w))
    assert w9[h] == pytest.approx(w[h] / 2) and w9[7] == pytest.approx(w[h] / 2)
    np.testing.assert_allclose(x9[7], y[h], atol=0)
