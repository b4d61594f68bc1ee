"""GPU (CUDA path through the C ABI) vs fp64 oracle parity, north_star tolerances:
  fp64, after one iteration (+ support update): Pi/w/x within 1e-10 relative (hybrid floor 1e-14*max)
  fp32, after one iteration:                      within 1e-5 relative (hybrid)
  fp32, after the full schedule:                  objective 1e-3 rel, w 1e-4 abs, x 1e-3 rel
Both sides read the same seeded bundle (paper_1510_00012_b200.workloads) with the same labels
and initial centroids, cluster by cluster.
"""
import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import workloads as wl
from paper_1510_00012_b200 import ad2
from tests.harness import run_gpu, assert_hybrid

pytestmark = pytest.mark.gpu


def compare_round(b, T, tau, rule=0, *, rtol_plan, rtol_x, atol_w, rtol_obj=None, check_plans=True, ctx=None,
                  mem="device", nccl=False, clusters=None, floor=1e-4):
    ctx, rho, obj = run_gpu(b, T, tau, rule, mem=mem, nccl=nccl, ctx=ctx)
    ores, members = oracle.run_bundle(b, T=T, tau=tau, rule=rule, clusters=clusters, want_state=check_plans)
    x, w = ctx.centroids()
    mats = {}
    if check_plans:
        mats = {n: ctx.member_matrices(wch) for n, wch in (("Pi1", ad2.PI1), ("Pi2", ad2.PI2), ("Lam", ad2.LAMBDA))}
    for c, r in ores.items():
        assert rho[c] == pytest.approx(r.rho, rel=1e-12 if b.dtype == "f64" else 1e-6)
        assert np.abs(w[c] - r.w).max() <= atol_w, f"w cluster {c}: {np.abs(w[c] - r.w).max()}"
        assert_hybrid(x[c], r.x, rtol_x, floor=1.0, what=f"x cluster {c}")
        if rtol_obj is not None:
            # relative, with a floor of rtol_obj/100 x the cluster's mean entry cost (rho / rho0, X1):
            # the working-precision cost has an absolute error on the data's scale, which decides
            # clusters whose objective is ~0 (a single member is its own barycenter, P6)
            floor = rtol_obj * 1e-2 * r.rho / b.sched.rho0
            assert abs(obj[c] - r.obj) <= rtol_obj * abs(r.obj) + floor, f"objective cluster {c}: {obj[c]} {r.obj}"
        if check_plans:
            for name in ("Pi1", "Pi2"):
                got = np.concatenate([mats[name][k].ravel() for k in members[c]])
                want = np.concatenate([M.ravel() for M in r.mats[name]])
                assert_hybrid(got, want, rtol_plan, floor=floor, what=f"{name} cluster {c}")
            # Lambda = rho * (accumulated difference of nearly equal plans): compare on rho's scale
            got = np.concatenate([mats["Lam"][k].ravel() for k in members[c]])
            want = np.concatenate([M.ravel() for M in r.mats["Lam"]])
            assert np.abs(got - want).max() <= rtol_plan * r.rho * max(1.0, np.abs(want).max() / r.rho) * 10
    return ctx, ores


# ------------------------------------------------------------------ fp64, one iteration, 1e-10

def test_cfg1_fp64_one_iteration():
    b = wl.make_config(1)
    compare_round(b, T=1, tau=1, rtol_plan=1e-10, rtol_x=1e-10, atol_w=1e-12, floor=1e-4)


@pytest.mark.parametrize("rule", [0, 1])
def test_cfg1_fp64_full_schedule(rule):
    b = wl.make_config(1)
    compare_round(b, T=100, tau=20, rule=rule, rtol_plan=1e-8, rtol_x=1e-9, atol_w=1e-10, rtol_obj=1e-9)


@pytest.mark.parametrize("m,mk,d", [(5, (1, 9), 3), (16, (1, 16), 2), (13, (20, 30), 4), (40, (1, 12), 3),
                                    (64, (20, 64), 5)])
def test_fp64_ragged_shapes_one_and_five_iterations(m, mk, d):
    """Ragged m_k (incl. m_k = 1), m not a power of two, the two-chunk and generic kernels."""
    b = wl.make_random(300, m, d, K=3, mk_range=mk, seed=m, dtype="f64", T=1, tau=1)
    compare_round(b, T=1, tau=1, rtol_plan=1e-10, rtol_x=1e-10, atol_w=1e-12)
    compare_round(b, T=5, tau=2, rtol_plan=1e-9, rtol_x=1e-9, atol_w=1e-11, rtol_obj=1e-9)


@pytest.mark.parametrize("m,mk,d", [(32, (1, 32), 3), (24, (3, 29), 16)])
def test_fp64_32_row_blocks_step_shapes(m, mk, d):
    """32-row blocks (pair layout, odd and even m_k): steps of 1 (P2X), 2 and 3 (FUSEDX) and a
    trailing single step, with the deferred phase 2 stored on read-back, vs the oracle in fp64."""
    b = wl.make_random(240, m, d, K=3, mk_range=mk, seed=100 + m, dtype="f64", T=1, tau=1)
    ctx, _ = compare_round(b, T=1, tau=1, rtol_plan=1e-10, rtol_x=1e-10, atol_w=1e-12)
    info = ctx.info()
    assert (info["variant"], info["mp"]) == (2, 32), info
    compare_round(b, T=5, tau=2, rtol_plan=1e-9, rtol_x=1e-9, atol_w=1e-11, rtol_obj=1e-9)
    compare_round(b, T=9, tau=3, rtol_plan=1e-9, rtol_x=1e-9, atol_w=1e-11, rtol_obj=1e-9)


# ------------------------------------------------------------------ fp32

@pytest.mark.parametrize("m,mk,d", [(64, (20, 64), 64), (48, (1, 64), 24), (40, (5, 33), 64)])
def test_fp32_warp_pair_step_shapes(m, mk, d):
    """The cached-cost warp-pair kernel (variant 3): a cold round's P1INIT pass (Pi2^0, Lambda = 0
    formed in the pass), steps of 2 and 3 ending with FUSEDX (support-update partials from the
    supports staged into the consumed C slot, phase 2 deferred), a step of 1 (P2X), and the
    deferred phase 2 stored on read-back, against the oracle (fp32 after a few iterations: plans
    within 1e-4 relative, x within 1e-4, w within 1e-5)."""
    b = wl.make_random(300, m, d, K=3, mk_range=mk, seed=300 + m + d, dtype="f32", T=1, tau=1, spread=2.0)
    ctx, _ = compare_round(b, T=2, tau=2, rtol_plan=1e-4, rtol_x=1e-4, atol_w=1e-5)
    assert ctx.info()["variant"] == 3, ctx.info()
    compare_round(b, T=6, tau=3, rtol_plan=1e-4, rtol_x=1e-4, atol_w=1e-5, rtol_obj=1e-4)
    compare_round(b, T=5, tau=2, rtol_plan=1e-4, rtol_x=1e-4, atol_w=1e-5, rtol_obj=1e-4)


@pytest.mark.parametrize("cfg,N", [(2, 2000), (3, 2000), (5, 3000), (4, 1500)])
def test_fp32_one_iteration(cfg, N):
    b = wl.make_config(cfg, N=N)
    compare_round(b, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6)


@pytest.mark.parametrize("cfg,N", [(2, 2000), (3, 2000), (5, 3000), (4, 1500)])
def test_fp32_full_schedule(cfg, N):
    b = wl.make_config(cfg, N=N)
    compare_round(b, T=b.sched.T, tau=b.sched.tau, rtol_plan=None, rtol_x=1e-3, atol_w=1e-4, rtol_obj=1e-3,
                  check_plans=False)


def test_fp32_r2_rule():
    b = wl.make_config(3, N=1500, K=6)
    compare_round(b, T=1, tau=1, rule=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6)
    compare_round(b, T=30, tau=10, rule=1, rtol_plan=None, rtol_x=1e-3, atol_w=1e-4, rtol_obj=1e-3,
                  check_plans=False)


def expected_variant(m, mkmax, d, dtype="f32"):
    fits = [mp for mp in (8, 16, 32) if m <= mp and mkmax <= (32 if mp == 32 else 2 * mp)]
    if fits and d <= 16:
        return 2
    if dtype == "f32" and m <= 128 and mkmax <= 128:    # any d (d > 64: external x partials)
        return 3
    return 0


@pytest.mark.parametrize("m,mk,d", [(6, (1, 40), 2), (32, (30, 64), 16), (48, (4, 32), 16), (8, (1, 16), 3),
                                    (12, (10, 32), 5), (20, (1, 32), 7), (32, (1, 4), 16), (3, (1, 3), 1),
                                    (64, (20, 64), 64), (64, (1, 64), 5), (33, (1, 63), 9), (64, (1, 3), 64),
                                    (40, (60, 64), 64), (64, (1, 80), 3), (32, (1, 64), 32), (16, (1, 30), 24),
                                    (20, (30, 64), 5), (32, (10, 20), 64), (48, (4, 40), 130), (64, (20, 64), 100),
                                    (20, (1, 50), 300), (100, (20, 64), 5), (96, (1, 40), 300), (128, (10, 64), 16),
                                    (100, (50, 100), 300), (64, (60, 128), 16), (20, (1, 120), 3), (8, (100, 140), 2)])
def test_fp32_ragged_shapes(m, mk, d):
    """Covers the TMA kernel's G = 4 / 2 / 1 member packings, padded rows (m < MP), the
    two-chunk column sums, tiny m_k, the cached-cost warp-group kernel (one warp per member for
    m <= 32, a pair for m <= 64, four warps for m <= 128; m_k up to 128; any d, with the external
    x partials for d > 64), and the generic kernel (m_k > 128)."""
    b = wl.make_random(500, m, d, K=4, mk_range=mk, seed=7 + m, dtype="f32", T=1, tau=1)
    ctx, _ = compare_round(b, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6)
    v = expected_variant(m, int(b.sizes.max()), d)
    assert ctx.info()["variant"] == v
    if v == 3:                                        # one warp per member (ld 32) or a warp pair (ld 64)
        assert ctx.info()["mp"] == (32 if m <= 32 else (64 if m <= 64 else 128))
    compare_round(b, T=12, tau=4, rtol_plan=None, rtol_x=1e-3, atol_w=1e-4, rtol_obj=1e-3, check_plans=False)


# ------------------------------------------------------------------ tensor-core cost build (config 4)

def test_tc_bf16_cost_build_cfg4():
    """cost_mode 1 (tcgen05, bf16 operands, fp32 accumulation) against the oracle's fp64 cost:
    |dC| <= 2^-7 |x_i||y_j| (bf16 rounding of both operands, Cauchy-Schwarz) + fp32 rounding;
    the fp32 build (cost_mode 0) is held to fp32 rounding only.  Partial 128-point tiles, m = 64."""
    b = wl.make_config(4, N=1500)
    sample = np.random.default_rng(1).choice(b.N, 200, replace=False)
    worst = {}
    for mode in (0, 1):
        ctx, _, _ = run_gpu(b, 0, 1, cost_mode=mode)
        assert ctx.info()["variant"] == 3
        Cg = ctx.member_matrices(ad2.COST)
        err = 0.0
        for k in sample:
            c = b.labels[k]
            Y = b.member(k)[0].astype(np.float64)
            x = b.x0[c].astype(np.float64)
            Co = oracle.cost(x, Y)
            nx, ny = np.linalg.norm(x, axis=1), np.linalg.norm(Y, axis=1)
            scale = nx[:, None] ** 2 + ny[None, :] ** 2
            bound = 4e-6 * scale + (2.0 ** -7 * nx[:, None] * ny[None, :] if mode == 1 else 0.0)
            d = np.abs(Cg[k].astype(np.float64) - Co)
            assert (d <= bound).all(), (mode, k, float((d - bound).max()))
            err = max(err, float(d.max()))
        worst[mode] = err
    assert worst[1] > worst[0]          # the tensor-core path really ran on bf16 operands
    # the whole schedule on the tensor-core cost stays close to the fp32 result (report-only bound)
    T, tau = b.sched.T, b.sched.tau
    ctx0, _, obj0 = run_gpu(b, T, tau, cost_mode=0)
    ctx1, _, obj1 = run_gpu(b, T, tau, cost_mode=1)
    assert np.isfinite(obj1).all()
    rel = np.abs(obj1 - obj0) / np.maximum(np.abs(obj0), 1e-3 * np.abs(obj0).max())
    assert np.median(rel) < 0.05, rel


def test_tc_cost_mode_rejected_without_cost_cache():
    b = wl.make_config(3, N=500, K=4)           # m = 32, d = 16: cost recomputed in-kernel
    with pytest.raises(ad2.AD2Error, match="ARG"):
        run_gpu(b, 0, 1, cost_mode=1)


# ------------------------------------------------------------------ paths that must agree exactly

def _state(ctx):
    x, w = ctx.centroids()
    return x, w, ctx.plans(ad2.PI1), ctx.plans(ad2.PI2), ctx.plans(ad2.LAMBDA), ctx.objective()


def test_host_batch_equals_device_batch():
    b = wl.make_config(3, N=1200, K=5)
    a = _state(run_gpu(b, 20, 10, mem="device")[0])
    h = _state(run_gpu(b, 20, 10, mem="host")[0])
    for u, v in zip(a, h):
        np.testing.assert_array_equal(u, v)


def test_nccl_single_rank_equals_local():
    b = wl.make_config(2, N=1500, K=4)
    a = _state(run_gpu(b, 20, 10)[0])
    n = _state(run_gpu(b, 20, 10, nccl=True)[0])
    for u, v in zip(a, n):
        np.testing.assert_array_equal(u, v)


def test_deterministic_rerun_and_profiling_does_not_change_results():
    b = wl.make_config(5, N=2000, K=8)
    a = _state(run_gpu(b, 20, 10)[0])
    c = _state(run_gpu(b, 20, 10, profile=True)[0])
    for u, v in zip(a, c):
        np.testing.assert_array_equal(u, v)


def test_member_order_does_not_matter_beyond_rounding():
    """Permuting the caller's members only changes the caller-order read-back (the library sorts
    by cluster with a stable counting sort, so the reduction order is unchanged)."""
    b = wl.make_config(3, N=1000, K=4)
    perm = np.random.default_rng(0).permutation(b.N)
    bp = b.subset(perm)
    x1, w1, *_ = _state(run_gpu(b, 10, 5)[0])
    x2, w2, *_ = _state(run_gpu(bp, 10, 5)[0])
    # stable sort keeps each cluster's relative member order -> not identical in general
    np.testing.assert_allclose(w1, w2, atol=1e-6)
    np.testing.assert_allclose(x1, x2, rtol=1e-5, atol=1e-5)


def test_warm_start_second_round():
    """Round 2 warm-starts Pi^(2) for members whose label is unchanged.  Each side
    carries its own round-1 state into round 2 (no oracle input comes from the GPU)."""
    b = wl.make_config(3, N=1200, K=5)
    warm = np.ones(b.N, np.uint8)
    warm[::3] = 0
    ctx, _, _ = run_gpu(b, 10, 5)
    x1, w1 = ctx.centroids()
    run_gpu(b, 10, 5, ctx=ctx, warm_mask=warm, x0=x1, w0=w1)
    x2, w2 = ctx.centroids()
    for c in range(b.K):
        mem = np.nonzero(b.labels == c)[0]
        sub = b.subset(mem)
        r1 = oracle.badmm_centroid(b.x0[c], b.w0[c], sub.offsets, sub.supports, sub.weights, 10, 5, 0, 2.0, 1e-16,
                                   1e-5)
        r2 = oracle.badmm_centroid(r1.x, r1.w, sub.offsets, sub.supports, sub.weights, 10, 5, 0, 2.0, 1e-16, 1e-5,
                                   warm=r1.mats["Pi2"], warm_mask=warm[mem])
        assert np.abs(w2[c] - r2.w).max() <= 1e-4
        assert_hybrid(x2[c], r2.x, 1e-3, floor=1.0, what=f"x c{c}")
        # a cold round 2 from the same centroids differs: the warm start is really used
        r2c = oracle.badmm_centroid(r1.x, r1.w, sub.offsets, sub.supports, sub.weights, 10, 5, 0, 2.0, 1e-16, 1e-5)
        assert np.abs(r2c.w - r2.w).max() > 1e-4


# ------------------------------------------------------------------ invariants at larger size

def test_invariants_cfg3_full_size():
    b = wl.make_config(3)
    ctx, rho, obj = run_gpu(b, 20, 10)
    x, w = ctx.centroids()
    assert np.abs(w.sum(1) - 1).max() < 1e-5 and (w >= 0).all()                       # P2
    P1 = ctx.member_matrices(ad2.PI1)
    P2 = ctx.member_matrices(ad2.PI2)
    L = ctx.member_matrices(ad2.LAMBDA)
    rng = np.random.default_rng(0)
    for k in rng.choice(b.N, 300, replace=False):
        c = b.labels[k]
        om = b.member(k)[1].astype(np.float64)
        np.testing.assert_allclose(P1[k].sum(0), om / om.sum(), rtol=2e-5, atol=1e-9)  # P1 columns
        np.testing.assert_allclose(P2[k].sum(1), w[c], rtol=2e-5, atol=1e-9)          # P1 rows
        assert abs(L[k].astype(np.float64).sum()) <= 1e-4 * rho[c]                     # P3
    assert np.isfinite(obj).all() and (obj > 0).all()


@pytest.mark.parametrize("cfg,clusters", [(3, [0, 37]), (4, [0, 61]), (5, [0, 201])])
def test_full_size_sampled_clusters(cfg, clusters):
    """Bench launch configuration at BASELINE.json's full size (configs 3, 4 and 5: the bench
    workload, 4M members); the oracle recomputes two sampled clusters over the whole schedule of
    one round.  north_star full-schedule tolerances (w 1e-4 abs, x 1e-3, objective 1e-3)."""
    b = wl.make_config(cfg)
    T, tau = b.sched.T, b.sched.tau
    ctx, rho, obj = run_gpu(b, T, tau)
    x, w = ctx.centroids()
    ores, _ = oracle.run_bundle(b, T=T, tau=tau, clusters=clusters, want_state=False)
    for c, r in ores.items():
        assert rho[c] == pytest.approx(r.rho, rel=1e-6)
        assert np.abs(w[c] - r.w).max() <= 1e-4
        assert_hybrid(x[c], r.x, 1e-3, floor=1.0, what=f"x c{c}")
        floor = 1e-5 * r.rho / b.sched.rho0
        assert abs(obj[c] - r.obj) <= 1e-3 * abs(r.obj) + floor, (c, obj[c], r.obj)
    ctx.close()


# ------------------------------------------------------------------ errors

def test_errors():
    import torch
    b = wl.make_random(10, 4, 2, K=3, mk_range=(2, 3), seed=1, dtype="f32")
    ctx = ad2.Context(0)
    with pytest.raises(ad2.AD2Error, match="STATE"):
        ctx.step(1)
    lab = b.labels.copy()
    lab[:] = 0                                                       # clusters 1, 2 empty
    with pytest.raises(ad2.AD2Error, match="EMPTY"):
        ctx.init(b.offsets, b.supports, b.weights, lab, b.x0, b.w0, 3, 4, mem="host")
    bad = b.weights.copy()
    bad[0] += 0.1
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.init(b.offsets, b.supports, bad, b.labels, b.x0, b.w0, 3, 4, mem="host")
    lab = b.labels.copy()
    lab[0] = 7
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.init(b.offsets, b.supports, b.weights, lab, b.x0, b.w0, 3, 4, mem="host")
    Y0 = np.zeros_like(b.supports)
    x0 = np.zeros_like(b.x0)
    with pytest.raises(ad2.AD2Error, match="ZERO_RHO"):
        ctx.init(b.offsets, Y0, b.weights, b.labels, x0, b.w0, 3, 4, mem="host")
    ctx.init(b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0, 3, 4, mem="host")
    with pytest.raises(ad2.AD2Error, match="STATE"):
        ctx.update_support()
    ctx.step(3)
    ctx.update_support()
    assert np.isfinite(ctx.objective()).all()
