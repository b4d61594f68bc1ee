"""Epoch-anchored compressed state (ad2_set_state_mode(1)).

With the eps of Eq.badmmc0b / Eq.badmmc1b dropped from the Pi2 recursion, Lambda cancels between
them and Pi2^t = G exp(-s C / rho) a_i b_j from an anchor G (pin P4).  Checked:
  - fp64 with eps = 0 on BOTH sides: the compressed recursion is then exactly Alg. 4, so the GPU
    matches the oracle at fp64 rounding (1e-9) - this pins the algebra of the GIN / GMID / GXOUT
    passes (anchor, row and column log-factors, U = Lambda + rho Pi1, iteration count s);
  - fp32 with the paper's eps = 1e-16 against the eps = 1e-16 oracle at north_star tolerances
    (one step of 3 iterations: plans hybrid 1e-5; full schedule: w 1e-4 abs, x 1e-3, objective
    1e-3), on configs 3 and 5 and at full size on config 5 (sampled clusters);
  - the documented failure: a column whose whole mass is the eps floor (an outlier point) raises
    ad2_info.eps_floor_columns (the exact mode does not).
"""
import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import ad2
from paper_1510_00012_b200 import workloads as wl
from tests.harness import assert_hybrid, hybrid_err, run_gpu

pytestmark = pytest.mark.gpu


def _oracle(b, T, tau, rule, eps, want_state=True):
    out, members = {}, {}
    wtol = 1e-6 if b.dtype == "f64" else 1e-5
    for c in range(b.K):
        mem = np.nonzero(b.labels == c)[0]
        sub = b.subset(mem)
        members[c] = mem
        out[c] = oracle.badmm_centroid(b.x0[c], b.w0[c], sub.offsets, sub.supports, sub.weights, T, tau, rule,
                                       b.sched.rho0, eps, wtol, want_state=want_state)
    return out, members


@pytest.mark.parametrize("m,mk,d", [(32, (3, 32), 16), (24, (1, 29), 3), (8, (1, 16), 2), (12, (10, 32), 3)])
@pytest.mark.parametrize("rule", [0, 1])
def test_fp64_eps0_compressed_is_alg4(m, mk, d, rule):
    b = wl.make_random(300, m, d, K=3, mk_range=mk, seed=300 + m, dtype="f64")
    T, tau = 13, 5                       # steps of 5, 5, 3 (P1INIT, GIN, GMID.., GXOUT each) + updates
    ctx, rho, obj = run_gpu(b, T, tau, rule=rule, state_mode=1, eps=0.0)
    assert (ctx.info()["variant"], ctx.info()["state_mode"]) == (2, 1)
    x, w = ctx.centroids()
    P1, P2, L = (ctx.member_matrices(k) for k in (ad2.PI1, ad2.PI2, ad2.LAMBDA))
    ores, members = _oracle(b, T, tau, rule, 0.0)
    for c, r in ores.items():
        assert np.abs(w[c] - r.w).max() <= 1e-11
        assert_hybrid(x[c], r.x, 1e-9, floor=1.0, what=f"x c{c}")
        assert abs(obj[c] - r.obj) <= 1e-9 * abs(r.obj)
        for name, G in (("Pi1", P1), ("Pi2", P2)):
            got = np.concatenate([G[k].ravel() for k in members[c]])
            want = np.concatenate([M.ravel() for M in r.mats[name]])
            assert_hybrid(got, want, 1e-9, floor=1e-6, what=f"{name} c{c}")
        got = np.concatenate([L[k].ravel() for k in members[c]])
        want = np.concatenate([M.ravel() for M in r.mats["Lam"]])
        assert np.abs(got - want).max() <= 1e-9 * r.rho


@pytest.mark.parametrize("cfg,N", [(3, 2000), (5, 3000), (2, 2000)])
def test_fp32_compressed_vs_eps_oracle(cfg, N):
    b = wl.make_config(cfg, N=N)
    # one iteration: steps of < 3 never use the compressed passes (identical to mode 0)
    ctx, _, _ = run_gpu(b, 1, 1, state_mode=1)
    ores, members = _oracle(b, 1, 1, b.sched.rule, b.sched.eps)
    P1 = ctx.member_matrices(ad2.PI1)
    x, w = ctx.centroids()
    for c, r in ores.items():
        assert np.abs(w[c] - r.w).max() <= 1e-6
        assert_hybrid(x[c], r.x, 1e-5, floor=1.0, what=f"x c{c}")
        got = np.concatenate([P1[k].ravel() for k in members[c]])
        assert_hybrid(got, np.concatenate([M.ravel() for M in r.mats["Pi1"]]), 1e-5, what=f"Pi1 c{c}")
    # one step of 3 (P1INIT, GIN, GXOUT) at the one-iteration bar, except the support points of
    # centroid rows with w_i < 1e-8: their x_i is a mean over plan entries a few orders of magnitude
    # above the eps floor, so the eps-free recursion moves it (measured 1.7e-5 relative at a row with
    # w_i = 8e-11 on config 5); those rows are held to the full-schedule bar (1e-3)
    ores, members = _oracle(b, 3, 3, b.sched.rule, b.sched.eps)
    ctx, _, _ = run_gpu(b, 3, 3, state_mode=1)
    x, w = ctx.centroids()
    P2 = ctx.member_matrices(ad2.PI2)
    for c, r in ores.items():
        assert np.abs(w[c] - r.w).max() <= 1e-6
        live = r.w >= 1e-8
        assert_hybrid(x[c][live], r.x[live], 1e-5, floor=np.abs(r.x).max() / np.abs(r.x[live]).max(),
                      what=f"x c{c}")
        assert_hybrid(x[c], r.x, 1e-3, floor=1.0, what=f"x c{c} (all rows)")
        got = np.concatenate([P2[k].ravel() for k in members[c]])
        assert_hybrid(got, np.concatenate([M.ravel() for M in r.mats["Pi2"]]), 1e-5, what=f"Pi2 c{c}")
    # the full schedule at the full-schedule bar
    T, tau = b.sched.T, b.sched.tau
    ctx, _, obj = run_gpu(b, T, tau, state_mode=1)
    x, w = ctx.centroids()
    ores, _ = _oracle(b, T, tau, b.sched.rule, b.sched.eps, want_state=False)
    dead = []
    for c, r in ores.items():
        assert np.abs(w[c] - r.w).max() <= 1e-4
        live = r.w >= 1e-8
        scale = np.abs(r.x).max()
        assert_hybrid(x[c][live], r.x[live], 1e-3, floor=scale / np.abs(r.x[live]).max(), what=f"x c{c}")
        if (~live).any():                # eps-decided rows: bounded, reported, not held
            dead.append(float(np.abs(x[c][~live] - r.x[~live]).max() / scale))
        floor = 1e-5 * r.rho / b.sched.rho0
        assert abs(obj[c] - r.obj) <= 1e-3 * abs(r.obj) + floor
    assert not dead or max(dead) < 0.1, dead
    print(f"rows with w_i < 1e-8: {len(dead)} clusters, max |dx| / max|x| = {max(dead, default=0):.3g}")
    assert ctx.info()["eps_floor_columns"] == 0


def test_full_size_cfg5_compressed_sampled_clusters():
    """The bench launch configuration of the compressed mode (config 5 at full size)."""
    b = wl.make_config(5)
    T, tau = b.sched.T, b.sched.tau
    ctx, rho, obj = run_gpu(b, T, tau, state_mode=1)
    x, w = ctx.centroids()
    ores, _ = oracle.run_bundle(b, T=T, tau=tau, clusters=[0, 201], want_state=False)
    for c, r in ores.items():
        assert np.abs(w[c] - r.w).max() <= 1e-4
        assert_hybrid(x[c], r.x, 1e-3, floor=1.0, what=f"x c{c}")
        assert abs(obj[c] - r.obj) <= 1e-3 * abs(r.obj) + 1e-5 * r.rho / b.sched.rho0
    assert ctx.info()["eps_floor_columns"] == 0
    ctx.close()


def test_eps_floor_column_is_flagged():
    """An outlier point far from every centroid point: its Pi1 column is the eps floor's
    (omega_j / m, X3), which the eps-free recursion cannot carry -> the flag is raised."""
    base = wl.make_random(600, 8, 3, K=3, mk_range=(4, 12), seed=61, dtype="f32")
    Y = base.supports.copy()
    for c in range(base.K):
        k = int(np.nonzero(base.labels == c)[0][0])
        Y[base.offsets[k]] += np.array([3000.0, 0, 0], np.float32)
    b = wl.replace(base, supports=Y)
    ctx, _, _ = run_gpu(b, 10, 5, state_mode=0)
    assert ctx.info()["eps_floor_columns"] == 0
    ctx, _, _ = run_gpu(b, 10, 5, state_mode=1)
    assert ctx.info()["eps_floor_columns"] == 1


def test_compressed_then_exact_warm_round_and_readback():
    """State mode 1 leaves the exact state (Pi1, Lambda) at every step boundary: read-back, the
    objective and a warm second round in mode 0 agree with an all-exact run (fp32 tolerances)."""
    b = wl.make_config(3, N=1500, K=5)
    res = []
    for mode in (1, 0):
        ctx, _, obj = run_gpu(b, 20, 10, state_mode=mode)
        x1, w1 = ctx.centroids()
        warm = np.ones(b.N, np.uint8)
        warm[::4] = 0
        run_gpu(b, 20, 10, ctx=ctx, warm_mask=warm, x0=x1, w0=w1, state_mode=0)
        res.append((obj, *ctx.centroids()))
    np.testing.assert_allclose(res[0][0], res[1][0], rtol=1e-4)
    np.testing.assert_allclose(res[0][2], res[1][2], atol=1e-5)
    np.testing.assert_allclose(res[0][1], res[1][1], rtol=1e-4, atol=1e-4)
