"""Symbolic-support mode: cost from a symbol-to-symbol table,
support update skipped.  GPU (cost_mode = AD2_COST_TABLE through the C ABI) vs the oracle's
``badmm_table`` on the same seeded symbolic bundle, cluster by cluster, with the north_star
tolerances (fp64 one iteration 1e-10; fp32 one iteration 1e-5; fp32 full schedule w 1e-4 abs,
objective 1e-3 rel), and the symbolic assignment vs exact transport on the table costs."""
import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import ad2, workloads as wl
from tests.harness import assert_hybrid, torch_cuda

pytestmark = pytest.mark.gpu


def run_sym(b, T, mem="device"):
    torch = torch_cuda()
    ctx = ad2.Context(0)
    ctx.set_cost_table(b.D)
    if mem == "device":
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        args = [t(b.offsets), t(b.ids), t(b.weights), t(b.labels), t(b.xs0), t(b.w0)]
    else:
        args = [b.offsets, b.ids, b.weights, b.labels, b.xs0, b.w0]
    rho = ctx.init(*args, b.K, b.m, 2.0, 1e-16, 0, mem=mem, dtype=b.dtype, cost_mode=ad2.COST_TABLE)
    ad2.run_schedule(ctx, T, b.sched.tau)
    obj = ctx.objective()
    return ctx, rho, obj


def oracle_sym(b, c, T):
    mem = np.nonzero(b.labels == c)[0]
    off = np.concatenate([[0], np.cumsum(np.diff(b.offsets)[mem])]).astype(np.int64)
    ids = np.concatenate([b.ids[b.offsets[k]:b.offsets[k + 1]] for k in mem])
    om = np.concatenate([b.weights[b.offsets[k]:b.offsets[k + 1]] for k in mem]).astype(np.float64)
    wtol = 1e-6 if b.dtype == "f64" else 1e-5
    return oracle.badmm_table(b.xs0[c], b.w0[c], off, ids, om, b.D, T, wtol=wtol), mem


@pytest.mark.parametrize("dtype,m,rtol", [("f32", 16, 1e-5), ("f32", 48, 1e-5), ("f64", 16, 1e-10)])
def test_symbolic_one_iteration(dtype, m, rtol):
    b = wl.make_symbolic(N=300, K=4, m=m, dtype=dtype)
    ctx, rho, obj = run_sym(b, 1)
    assert ctx.info()["variant"] == (3 if dtype == "f32" else 0)
    xs, w = ctx.centroids()
    np.testing.assert_array_equal(xs, b.xs0)                      # symbols are never updated
    P1 = ctx.member_matrices(ad2.PI1)
    for c in range(b.K):
        r, mem = oracle_sym(b, c, 1)
        assert rho[c] == pytest.approx(r.rho, rel=1e-12 if dtype == "f64" else 1e-6)
        np.testing.assert_allclose(w[c], r.w, rtol=rtol, atol=rtol * 1e-3)
        got = np.concatenate([P1[k].ravel() for k in mem])
        want = np.concatenate([M.ravel() for M in r.mats["Pi1"]])
        assert_hybrid(got, want, rtol, floor=1e-4, what=f"Pi1 c{c}")


@pytest.mark.parametrize("mem", ["device", "host"])
def test_symbolic_full_schedule_fp32(mem):
    b = wl.make_symbolic(N=400, K=5, m=16)
    T = b.sched.T
    ctx, rho, obj = run_sym(b, T, mem=mem)
    _, w = ctx.centroids()
    for c in range(b.K):
        r, _ = oracle_sym(b, c, T)
        assert np.abs(w[c] - r.w).max() <= 1e-4
        assert abs(obj[c] - r.obj) <= 1e-3 * abs(r.obj) + 1e-5 * r.rho / 2.0


def test_symbolic_assignment_matches_exact_transport():
    b = wl.make_symbolic(N=150, K=4, m=12, dtype="f64")
    ctx = ad2.Context(0)
    ctx.set_cost_table(b.D)
    lab, w2, n_exact = ctx.assign_symbolic(b.offsets, b.ids, b.weights, b.xs0, b.w0, mem="host")
    for k in range(b.N):
        ids = b.ids[b.offsets[k]:b.offsets[k + 1]]
        om = b.weights[b.offsets[k]:b.offsets[k + 1]]
        W = np.array([oracle.transport(b.w0[c] / b.w0[c].sum(), om / om.sum(), b.D[np.ix_(b.xs0[c], ids)])
                      for c in range(b.K)])
        srt = np.sort(W)
        if srt[1] - srt[0] > 1e-6:
            assert lab[k] == int(np.argmin(W)), k
        assert w2[k] == pytest.approx(W.min(), rel=1e-9, abs=1e-12)


def test_symbolic_cluster_loop():
    b = wl.make_symbolic(N=500, K=4, m=16)
    torch = torch_cuda()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ctx = ad2.Context(0)
    ctx.set_cost_table(b.D)
    res = ctx.cluster(t(b.offsets), t(b.ids), t(b.weights), t(b.labels), t(b.xs0), t(b.w0), b.K, b.m, 20, 10, 4,
                      cost_mode=ad2.COST_TABLE)
    assert res["rounds"] >= 1 and np.isfinite(res["objective"]).all()
    xs, w = ctx.centroids()
    np.testing.assert_array_equal(xs, b.xs0)
    lab, _, _ = ctx.assign_symbolic(t(b.offsets), t(b.ids), t(b.weights), t(xs), t(w))
    np.testing.assert_array_equal(lab, res["labels"])


def test_symbolic_bad_ids_rejected():
    b = wl.make_symbolic(N=50, K=2, m=8)
    ids = b.ids.copy()
    ids[3] = b.V + 5
    ctx = ad2.Context(0)
    ctx.set_cost_table(b.D)
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.init(b.offsets, ids, b.weights, b.labels, b.xs0, b.w0, b.K, b.m, mem="host", dtype="f32",
                 cost_mode=ad2.COST_TABLE)
