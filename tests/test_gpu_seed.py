"""GPU initial partition (ad2_kmeanspp / ad2_label_nearest / ad2_pick_members, SURVEY.md §8(f)
NEXT #2) vs the oracle (oracle/seed.py) on the same draws.

Every index here is decided by fp64 arithmetic that both sides evaluate in the same order
(X21: distances, member means, Lloyd sums in index order), except the D^2 draw's prefix
sum (X20: blocked on the GPU, sequential in the oracle), which can move a draw only when
u * sum D^2 lands within rounding of a prefix boundary.  So the bar is bit-exact: centres, labels
and picks equal element by element.
"""
import numpy as np
import pytest

from oracle import seed
from paper_1510_00012_b200 import workloads as wl
from tests.harness import to_dev, torch_cuda

pytestmark = pytest.mark.gpu


def draws(N, K, ns, s=0):
    rng = np.random.default_rng([11, s, N, K])
    return rng.choice(N, size=ns, replace=False), rng.uniform(size=K), rng.uniform(size=K)


def run_both(b, K, ns, iters=10, mem="device", s=0):
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    sample, u, up = draws(b.N, K, ns, s)
    ctx = ad2.Context(0)
    if mem == "device":
        a = to_dev(b, torch)
        off, Y, W = a["offsets"], a["supports"], a["weights"]
    else:
        off, Y, W = b.offsets, b.supports, b.weights
    cen = ctx.kmeanspp(off, Y, W, sample, u, iters, mem=mem, dtype=b.dtype)
    ocen = seed.kmeanspp(seed.member_means(b.offsets, b.supports, b.weights)[sample], K, u, iters)
    assert np.array_equal(cen, ocen), np.abs(cen - ocen).max()
    lab, cen2 = ctx.label_nearest(off, Y, W, cen, mem=mem, dtype=b.dtype)
    olab, ocen2 = seed.label_nearest(seed.member_means(b.offsets, b.supports, b.weights), ocen)
    assert np.array_equal(lab, olab), np.count_nonzero(lab != olab)
    assert np.array_equal(cen2, ocen2)
    if mem == "device":
        labd = torch.from_numpy(lab).cuda()
    else:
        labd = lab
    pick = ctx.pick_members(off, Y, W, labd, b.m, up, mem=mem, dtype=b.dtype)
    assert np.array_equal(pick, seed.pick_members(b.offsets, lab, b.m, up))
    ctx.close()
    return lab, pick


@pytest.mark.parametrize("cfg,N,K,ns", [(2, 20_000, 10, 2_000), (3, 30_000, 64, 3_000), (4, 20_000, 100, 2_000),
                                        (5, 60_000, 256, 6_000)])
def test_partition_matches_oracle(cfg, N, K, ns):
    b = wl.make_config(cfg, N=N, K=K)
    lab, pick = run_both(b, K, ns)
    assert np.bincount(lab, minlength=K).min() >= 1
    sizes = np.diff(b.offsets)
    assert np.all(lab[pick] == np.arange(K))
    assert np.all((sizes[pick] >= b.m) | (np.bincount(lab, weights=(sizes >= b.m), minlength=K)[np.arange(K)] == 0))


def test_partition_full_size_cfg3():
    """config 3 at its full size (N = 200k, the 10 % sample of SURVEY.md §8(d), K = 64)."""
    b = wl.make_config(3, K=64)
    run_both(b, 64, 20_000, s=1)


def test_partition_host_batch_fp64():
    b = wl.make_config(1, N=200)
    run_both(b, 3, 50, iters=5, mem="host")


def test_partition_wide_d_and_ragged():
    """d = 40 and d = 130 (two and five coordinates per lane), ns not a multiple of the 256-point
    D^2 block, K not a multiple of the warps per block."""
    for d, N, K, ns in ((40, 3_001, 7, 777), (130, 1_500, 5, 513)):
        rng = np.random.default_rng(d)
        sizes = rng.integers(1, 9, size=N)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        Y = (rng.normal(size=(off[-1], d)) + rng.integers(0, 4, size=(off[-1], 1)) * 3.0).astype(np.float32)
        W = rng.dirichlet(np.ones(8), size=N)
        Wf = np.concatenate([W[k, :sizes[k]] / W[k, :sizes[k]].sum() for k in range(N)]).astype(np.float32)
        b = wl.Bundle("rand", d, 4, K, off, Y, Wf, np.zeros(N, np.int32), np.zeros((K, 4, d)), np.zeros((K, 4)),
                      "f32", None)
        run_both(b, K, ns, iters=4)


def test_empty_cluster_repair_matches_oracle():
    """centres far from every member leave clusters empty: the repair (X22) on both sides."""
    from paper_1510_00012_b200 import ad2
    b = wl.make_config(2, N=5_000, K=10)
    mu = seed.member_means(b.offsets, b.supports, b.weights)
    cen = np.concatenate([mu[:4], np.full((4, 3), 1e3), mu[4:6]])
    ctx = ad2.Context(0)
    lab, cen2 = ctx.label_nearest(b.offsets, b.supports, b.weights, cen, mem="host", dtype=b.dtype)
    olab, ocen2 = seed.label_nearest(mu, cen)
    assert np.array_equal(lab, olab) and np.array_equal(cen2, ocen2)
    assert np.bincount(lab, minlength=10).min() >= 1
    ctx.close()


def test_equal_means_take_uniform_draws():
    """every member mean equal: D^2 = 0 after the first centre, draws fall back to floor(u ns)."""
    from paper_1510_00012_b200 import ad2
    N, K = 600, 6
    off = np.arange(N + 1, dtype=np.int64)
    Y = np.full((N, 2), 0.25)
    W = np.ones(N)
    sample, u, _ = draws(N, K, 300)
    ctx = ad2.Context(0)
    cen = ctx.kmeanspp(off, Y, W, sample, u, 3, mem="host", dtype="f64")
    assert np.array_equal(cen, seed.kmeanspp(np.full((300, 2), 0.25), K, u, 3))
    lab, _ = ctx.label_nearest(off, Y, W, cen, mem="host", dtype="f64")
    olab, _ = seed.label_nearest(np.full((N, 2), 0.25), cen)
    assert np.array_equal(lab, olab)
    ctx.close()


def test_partition_argument_errors():
    from paper_1510_00012_b200 import ad2
    b = wl.make_config(2, N=500, K=5)
    ctx = ad2.Context(0)
    args = (b.offsets, b.supports, b.weights)
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.kmeanspp(*args, np.array([0, 1, 500, 3, 4, 5]), np.full(5, 0.5), 1, mem="host")
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.kmeanspp(*args, np.arange(10), np.array([0.1, 0.2, 1.0, 0.3, 0.4]), 1, mem="host")
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ctx.kmeanspp(*args, np.arange(3), np.full(5, 0.5), 1, mem="host")          # ns < K
    with pytest.raises(ad2.AD2Error, match="EMPTY"):
        ctx.pick_members(*args, np.zeros(500, np.int32), b.m, np.full(5, 0.5), mem="host")
    ctx.close()


def test_partition_edge_shapes():
    """ns = K (every sampled mean becomes a centre), d = 256 (the largest d), one-point members."""
    for d, N, K, ns in ((5, 400, 8, 8), (256, 300, 4, 40), (1, 500, 3, 3)):
        rng = np.random.default_rng(100 + d)
        sizes = rng.integers(1, 4, size=N) if d != 1 else np.ones(N, np.int64)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        Y = rng.normal(size=(off[-1], d)) * 3.0
        Wf = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
        b = wl.Bundle("edge", d, 2, K, off, Y, Wf, np.zeros(N, np.int32), np.zeros((K, 2, d)), np.zeros((K, 2)),
                      "f64", None)
        lab, pick = run_both(b, K, ns, iters=3, mem="host")
        if ns == K:                                   # distinct means: every sampled mean is a centre
            assert len(np.unique(lab)) == K
