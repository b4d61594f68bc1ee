"""GPU assignment step (ad2_assign) vs the oracle's exact-OT assignment
(oracle.assign: transportation simplex against every centroid, lowest index on ties).

north_star: labels bit-exact wherever the oracle's distance gap (second-best - best W^2) exceeds
1e-6, compared on IDENTICAL centroids (both sides get the same x, w).  The minimum W^2 itself is
an exact LP optimum on both sides (fp64), so it must agree to fp64 rounding: 1e-9 relative.
"""
import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import workloads as wl
from tests.harness import run_gpu, to_dev, torch_cuda

pytestmark = pytest.mark.gpu


def check_assign(b, x, w, mem="device"):
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    ctx = ad2.Context(0)
    if mem == "device":
        a = to_dev(b, torch)
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
        lab, w2, n_exact = ctx.assign(a["offsets"], a["supports"], a["weights"], xd, wd, dtype=b.dtype)
    else:
        lab, w2, n_exact = ctx.assign(b.offsets, b.supports, b.weights, np.ascontiguousarray(x),
                                      np.ascontiguousarray(w), mem="host", dtype=b.dtype)
    olab, obest, osecond = oracle.assign(x, w, b.offsets, b.supports, b.weights)
    gap = osecond - obest
    sure = gap > 1e-6
    assert (lab[sure] == olab[sure]).all(), np.nonzero(lab[sure] != olab[sure])
    # the GPU's W^2 is the exact minimum too
    np.testing.assert_allclose(w2, obest, rtol=1e-9, atol=1e-12 * max(1.0, float(np.abs(obest).max())))
    assert n_exact >= b.N if b.K > 1 else n_exact >= 0
    ctx.close()
    return lab, n_exact, sure


@pytest.mark.parametrize("cfg,N,K", [(2, 600, 10), (3, 300, 6), (5, 300, 8)])
def test_assign_initial_centroids(cfg, N, K):
    b = wl.make_config(cfg, N=N, K=K)
    lab, n_exact, sure = check_assign(b, b.x0, b.w0)
    assert sure.mean() > 0.9
    assert n_exact <= b.N * b.K                       # pruning never adds work


def test_assign_cfg4_host_batch():
    b = wl.make_config(4, N=120, K=5)
    check_assign(b, b.x0, b.w0, mem="host")


def test_assign_after_a_round_on_gpu_centroids():
    """The AD2 loop: B-ADMM round on the GPU, then labels against those (identical) centroids."""
    b = wl.make_config(2, N=800, K=6)
    ctx, _, _ = run_gpu(b, 20, 10)
    x, w = ctx.centroids()
    lab, n_exact, sure = check_assign(b, x, w)
    assert n_exact < b.N * b.K                        # the bounds prune on real clusters


@pytest.mark.parametrize("m,mk,d,K,dtype", [(5, (1, 9), 3, 7, "f64"), (3, (1, 1), 2, 4, "f32"),
                                             (6, (1, 12), 2, 1, "f64"), (33, (30, 40), 4, 3, "f32")])
def test_assign_ragged_and_edge_shapes(m, mk, d, K, dtype):
    b = wl.make_random(200, m, d, K=K, mk_range=mk, seed=3 + m, dtype=dtype)
    lab, _, _ = check_assign(b, b.x0, b.w0)
    if K == 1:
        assert (lab == 0).all()


@pytest.mark.parametrize("m,mk,d,K,dtype", [(100, (60, 128), 3, 3, "f32"),     # 4 nodes per lane and side
                                             (20, (120, 140), 2, 2, "f64")])    # m_k > 128: shared-memory SSP
def test_assign_large_supports(m, mk, d, K, dtype):
    b = wl.make_random(12, m, d, K=K, mk_range=mk, seed=11 + m, dtype=dtype)
    check_assign(b, b.x0, b.w0)


def test_assign_identity_and_duplicate_centroids():
    """Members equal to centroid c get c with W^2 = 0; a duplicated centroid ties to the lower index."""
    rng = np.random.default_rng(5)
    K, m, d = 5, 4, 3
    x = rng.normal(0, 4, (K, m, d))
    w = rng.dirichlet(np.ones(m), K)
    x[4], w[4] = x[2], w[2]
    off = np.arange(K + 1, dtype=np.int64) * m
    b = wl.Bundle("identity", d, m, K, off, x.reshape(-1, d).copy(), w.reshape(-1).copy(),
                  np.zeros(K, np.int32), x, w, "f64", wl.Schedule(T=1, tau=1))
    from paper_1510_00012_b200 import ad2
    ctx = ad2.Context(0)
    lab, w2, _ = ctx.assign(b.offsets, b.supports, b.weights, x, w, mem="host", dtype="f64")
    assert list(lab) == [0, 1, 2, 3, 2]
    assert np.abs(w2).max() < 1e-12


# ------------------------------------------------------------------ the outer loop (NEXT #2)

@pytest.mark.parametrize("mem", ["device", "host"])
def test_cluster_loop_fp64_matches_oracle_loop(mem):
    """ad2_cluster (fp64, 1e-10 parity per B-ADMM round) against the oracle's loop
    (oracle.cluster): identical labels every round (the gaps here are >> 1e-6), same rounds,
    changed fractions and objectives, and the final centroids."""
    from paper_1510_00012_b200 import ad2
    b = wl.make_config(3, N=240, K=4, dtype="f64")
    T, tau, R = 20, 10, 3
    olab, orounds, ochanged, oobj, ox, ow = oracle.cluster(b, T, tau, R)
    torch = torch_cuda()
    ctx = ad2.Context(0)
    if mem == "device":
        a = to_dev(b, torch)
        res = ctx.cluster(a["offsets"], a["supports"], a["weights"], a["labels"], a["x0"], a["w0"], b.K, b.m, T, tau,
                          R, dtype="f64")
    else:
        res = ctx.cluster(b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0, b.K, b.m, T, tau, R, mem="host",
                          dtype="f64")
    assert res["rounds"] == orounds
    np.testing.assert_array_equal(res["labels"], olab)
    np.testing.assert_allclose(res["changed"], ochanged, atol=0)
    np.testing.assert_allclose(res["objective"], oobj, rtol=1e-8)
    x, w = ctx.centroids()
    np.testing.assert_allclose(w, ow, atol=1e-10)
    np.testing.assert_allclose(x, ox, rtol=1e-8, atol=1e-9 * np.abs(ox).max())


def test_cluster_loop_fp32_stops_on_stable_labels():
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    b = wl.make_config(2, N=1500, K=5)
    a = to_dev(b, torch)
    ctx = ad2.Context(0)
    res = ctx.cluster(a["offsets"], a["supports"], a["weights"], a["labels"], a["x0"], a["w0"], b.K, b.m, 20, 10, 8,
                      stop_frac=0.01)
    ch = res["changed"]
    assert 1 <= res["rounds"] <= 8 and len(ch) == res["rounds"]
    assert res["rounds"] == 8 or ch[-1] <= 0.01
    assert np.isfinite(res["objective"]).all()
    # the returned labels are the exact assignment against the returned centroids
    x, w = ctx.centroids()
    lab, _, _ = ctx.assign(a["offsets"], a["supports"], a["weights"], torch.from_numpy(x).cuda(),
                           torch.from_numpy(w).cuda())
    np.testing.assert_array_equal(lab, res["labels"])


def _separated_groups(N=2000, K=6, m=8, d=3, seed=5, dtype="f32"):
    """K groups of distributions 60 units apart (members of a group scattered around its centre),
    initial labels with a fifth of the members mislabelled, centroids from a correct member each:
    the loop converges in a few rounds and later rounds move the centroids by << the gaps."""
    rng = np.random.default_rng(seed)
    truth = rng.integers(0, K, N).astype(np.int32)
    sizes = rng.integers(3, 12, N)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    centres = rng.normal(0, 60, (K, d))
    Y = np.repeat(centres[truth], sizes, axis=0) + rng.normal(0, 1.5, (off[-1], d))
    W = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
    lab0 = truth.copy()
    flip = rng.choice(N, N // 5, replace=False)
    lab0[flip] = rng.integers(0, K, len(flip))
    x0 = np.stack([centres[c] + rng.normal(0, 1.5, (m, d)) for c in range(K)])
    w0 = np.full((K, m), 1.0 / m)
    nt = np.float64 if dtype == "f64" else np.float32
    return wl.Bundle("separated", d, m, K, off, Y.astype(nt), W.astype(nt), lab0, x0.astype(nt), w0.astype(nt), dtype,
                     wl.Schedule(T=20, tau=10))


@pytest.mark.parametrize("case", ["cfg2", "cfg3", "cfg5", "separated"])
def test_cluster_pruning_keeps_every_label(case, monkeypatch):
    """Cross-round pruning of the loop's assignment (Elkan, with W = sqrt(W^2) a metric,
    P:855-862): the labels, rounds, changed fractions and objectives of every round are those of
    the unpruned loop, bit for bit, and the returned labels are the exact assignment against the
    returned centroids.  On well-separated groups later rounds certify members without a solve;
    on the BASELINE workloads the centroids' drift between rounds (W(Q_c^r, Q_c^r+1)) exceeds
    the members' best / second-best gaps many times, so few or none are certified."""
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    b = {"cfg2": lambda: wl.make_config(2, N=3000, K=10), "cfg3": lambda: wl.make_config(3, N=4000, K=16, dtype="f64"),
         "cfg5": lambda: wl.make_config(5, N=6000, K=24), "separated": _separated_groups}[case]()
    a = to_dev(b, torch)
    out = {}
    for prune in (False, True):
        if prune:
            monkeypatch.delenv("AD2_NO_PRUNE", raising=False)
        else:
            monkeypatch.setenv("AD2_NO_PRUNE", "1")
        ctx = ad2.Context(0)
        res = ctx.cluster(a["offsets"], a["supports"], a["weights"], a["labels"], a["x0"], a["w0"], b.K, b.m, 20, 10, 5,
                          dtype=b.dtype)
        out[prune] = (res, ctx.info(), ctx.centroids())
        ctx.close()
    r0, r1 = out[False][0], out[True][0]
    assert r0["rounds"] == r1["rounds"]
    np.testing.assert_array_equal(r0["labels"], r1["labels"])
    np.testing.assert_array_equal(r0["changed"], r1["changed"])
    np.testing.assert_array_equal(r0["objective"], r1["objective"])
    info, info0 = out[True][1], out[False][1]
    assert info0["assign_certified"] == 0
    print(f"{case}: rounds {r1['rounds']}, certified {info['assign_certified']} of {b.N * (r1['rounds'] - 1)} "
          f"member-rounds after round 1, exact solves {info['assign_exact']} vs {info0['assign_exact']} unpruned")
    if case == "separated":
        assert r1["rounds"] >= 2 and info["assign_certified"] > 0.25 * b.N * (r1["rounds"] - 1)
        assert info["assign_exact"] < info0["assign_exact"]
    x, w = out[True][2]
    ctx = ad2.Context(0)
    lab, _, _ = ctx.assign(a["offsets"], a["supports"], a["weights"], torch.from_numpy(x).cuda(),
                           torch.from_numpy(w).cuda(), dtype=b.dtype)
    np.testing.assert_array_equal(lab, r1["labels"])


# ------------------------------------------------------------------ Eq.merge initialisation

@pytest.mark.parametrize("cfg,N,K,dtype", [(2, 600, 10, "f32"), (3, 400, 6, "f64"), (4, 120, 5, "f32")])
def test_merge_init_matches_oracle(cfg, N, K, dtype):
    """ad2_merge_init (fp64 on the device, uncontracted operations in the oracle's order) against
    oracle.merge on the same picks: identical merge decisions, values to fp64 rounding (the cast
    to the batch dtype at the end)."""
    from paper_1510_00012_b200 import ad2
    b = wl.make_config(cfg, N=N, K=K, dtype=dtype)
    rng = np.random.default_rng(cfg)
    sizes = np.diff(b.offsets)
    pick = []
    for c in range(b.K):
        mem = np.nonzero(b.labels == c)[0]
        big = mem[sizes[mem] >= b.m]
        pick.append(int(rng.choice(big)) if len(big) else int(mem[0]))   # small members exercise the split
    ctx = ad2.Context(0)
    for mem_kind in ("host", "device"):
        if mem_kind == "device":
            a = to_dev(b, torch_cuda())
            x0, w0 = ctx.merge_init(a["offsets"], a["supports"], a["weights"], pick, b.K, b.m, dtype=dtype)
        else:
            x0, w0 = ctx.merge_init(b.offsets, b.supports, b.weights, pick, b.K, b.m, mem="host", dtype=dtype)
        for c, k in enumerate(pick):
            y, w = b.member(k)
            ox, ow = oracle.merge(y, w, b.m)
            tol = 1e-14 if dtype == "f64" else 1e-6
            np.testing.assert_allclose(w0[c], ow, rtol=tol, atol=tol * 1e-3)
            np.testing.assert_allclose(x0[c], ox, rtol=tol, atol=tol * np.abs(ox).max())


def test_next_row_api_errors():
    """Argument errors of the NEXT-row entry points are reported, not crashed on."""
    from paper_1510_00012_b200 import ad2
    b = wl.make_random(20, 4, 2, K=3, mk_range=(2, 5), seed=2, dtype="f32")
    ctx = ad2.Context(0)
    bad_off = b.offsets.copy()
    bad_off[3] = bad_off[2]                                   # a member with m_k = 0
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.assign(bad_off, b.supports, b.weights, b.x0, b.w0, mem="host")
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.merge_init(b.offsets, b.supports, b.weights, [0, 1, 99], b.K, b.m, mem="host")
    with pytest.raises(ad2.AD2Error, match="ARG"):              # loop parameters
        ctx.cluster(b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0, b.K, b.m, 0, 1, 1, mem="host")
    with pytest.raises(ad2.AD2Error, match="ARG"):              # symbolic round without a cost table
        ctx.init(b.offsets, np.zeros(int(b.offsets[-1]), np.int32), b.weights, b.labels,
                 np.zeros((b.K, b.m), np.int32), b.w0, b.K, b.m, mem="host", dtype="f32", cost_mode=ad2.COST_TABLE)
    # the context still works after the errors
    lab, w2, _ = ctx.assign(b.offsets, b.supports, b.weights, b.x0, b.w0, mem="host")
    assert (lab >= 0).all() and (lab < b.K).all() and np.isfinite(w2).all()


@pytest.mark.parametrize("cfg", [3, 5])
def test_assign_full_size_sampled_members(cfg):
    """The assignment at BASELINE.json's full size (config 3: N = 200k, K = 64; config 5: N = 4M,
    K = 256), where the pruning bounds meet many near-equal candidates; the oracle recomputes 300
    random members against every centroid (same x, w on both sides)."""
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    b = wl.make_config(cfg)
    ctx = ad2.Context(0)
    a = to_dev(b, torch)
    lab, w2, n_exact = ctx.assign(a["offsets"], a["supports"], a["weights"], a["x0"], a["w0"], dtype=b.dtype)
    ctx.close()
    sample = np.sort(np.random.default_rng(cfg).choice(b.N, 300, replace=False))
    sub = b.subset(sample)
    olab, obest, osecond = oracle.assign(b.x0, b.w0, sub.offsets, sub.supports, sub.weights)
    sure = (osecond - obest) > 1e-6
    assert sure.mean() > 0.8
    assert (lab[sample][sure] == olab[sure]).all()
    np.testing.assert_allclose(w2[sample], obest, rtol=1e-9, atol=1e-12 * float(np.abs(obest).max()))
