"""The member-sharded path of libad2 with 2 ranks on ONE GPU (PAPER.md
P:882-890: data divided into trunks that stay on their processor, the centroid update's sums
synchronised every iteration).  NCCL cannot put two ranks on one GPU, so the ranks are two
processes joined by the host process group (ad2_group_*): the same per-cluster partial sums, all-
reduced through shared memory inside the step graphs.  No kernel waits on another rank (the
exchange is a host-function node), so the two processes only time-share the GPU.  Correctness
only: these runs measure nothing ("unmeasured on hardware").

Each case runs the sharded schedule and compares with the unsharded run of the same bundle
(fp64: the partial sums only change order, 1e-12) and with the fp64 oracle (north_star: 1e-10
after one iteration + support update; 1e-9 over a schedule):
  - entry-balanced contiguous shards: every cluster split across the two ranks;
  - a rank owning no member of some cluster (its partial sums for that cluster are zero);
  - a rank with N = 0 (it still joins every collective);
  - errors agree across ranks: a bad label or off-simplex weights on ONE rank make BOTH ranks
    return an error instead of one rank waiting forever in the next collective.
"""
import multiprocessing as mp
import uuid

import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import workloads as wl
from paper_1510_00012_b200.sharding import shard_bounds
from tests.harness import assert_hybrid

pytestmark = pytest.mark.gpu


def _worker(name, world, rank, bundle, bounds, T, tau, faults, q):
    try:
        from paper_1510_00012_b200 import ad2
        ctx = ad2.Context(0)
        if world > 1:
            g = ad2.Group(name, world, rank, slot_bytes=1 << 20)
            ctx.attach_group(g)
        b = bundle.subset(np.arange(bounds[rank], bounds[rank + 1]))
        lab, wts = b.labels.copy(), b.weights.copy()
        if faults.get("label") == rank and b.N:
            lab[0] = b.K + 3
        if faults.get("weights") == rank and b.N:
            wts[0] += 0.3
        out = {}
        try:
            rho = ctx.init(b.offsets, b.supports, wts, lab, b.x0, b.w0, b.K, b.m, mem="host", dtype=bundle.dtype)
        except ad2.AD2Error as e:
            q.put((rank, {"error": e.status}))
            return
        out["rho"] = rho
        ad2.run_schedule(ctx, T, tau)
        out["obj"] = ctx.objective()
        out["x"], out["w"] = ctx.centroids()
        out["Pi1"] = ctx.member_matrices(ad2.PI1) if b.N else []
        out["Pi2"] = ctx.member_matrices(ad2.PI2) if b.N else []
        ctx.close()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, {"exc": traceback.format_exc()}))


def run_ranks(bundle, bounds, T, tau, faults=None, timeout=600):
    world = len(bounds) - 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/ad2d_{uuid.uuid4().hex[:12]}"
    ps = [ctx.Process(target=_worker, args=(name, world, r, bundle, bounds, T, tau, faults or {}, q))
          for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = dict(q.get(timeout=timeout) for _ in range(world))
    finally:
        for p in ps:
            p.join(60)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert "exc" not in res[r], res[r]["exc"]
    return res


def check_sharded(bundle, bounds, T, tau, rtol_oracle):
    one = run_ranks(bundle, np.array([0, bundle.N]), T, tau)[0]
    two = run_ranks(bundle, bounds, T, tau)
    # every rank holds the same all-reduced centroids, rho and objective (rank-order sums)
    for key in ("x", "w", "rho", "obj"):
        np.testing.assert_array_equal(two[0][key], two[1][key])
    # sharded vs unsharded: the partial sums only change order
    np.testing.assert_allclose(two[0]["w"], one["w"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(two[0]["x"], one["x"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(two[0]["rho"], one["rho"], rtol=1e-13)
    np.testing.assert_allclose(two[0]["obj"], one["obj"], rtol=1e-11)
    for r in range(2):
        for i, k in enumerate(range(bounds[r], bounds[r + 1])):
            np.testing.assert_allclose(two[r]["Pi1"][i], one["Pi1"][k], rtol=1e-10, atol=1e-18)
    # and against the oracle, cluster by cluster
    ores, members = oracle.run_bundle(bundle, T=T, tau=tau)
    for c, r in ores.items():
        assert np.abs(two[0]["w"][c] - r.w).max() <= rtol_oracle * 1e-2
        assert_hybrid(two[0]["x"][c], r.x, rtol_oracle, floor=1.0, what=f"x c{c}")
        assert abs(two[0]["obj"][c] - r.obj) <= rtol_oracle * abs(r.obj)
        for k, P in zip(members[c], r.mats["Pi2"]):
            rk = 0 if k < bounds[1] else 1
            assert_hybrid(two[rk]["Pi2"][k - bounds[rk]], P, rtol_oracle, what=f"Pi2 member {k}")
    return two


@pytest.mark.parametrize("shape", [(24, (3, 29), 3), (6, (1, 9), 2), (48, (20, 60), 5)])
def test_two_ranks_split_clusters(shape):
    m, mk, d = shape                    # variant 2 (pair layout), variant 2 (MP 8), generic fp64 kernel
    b = wl.make_random(400, m, d, K=3, mk_range=mk, seed=200 + m, dtype="f64")
    bounds = shard_bounds(b.offsets, 2)
    for c in range(b.K):                # every cluster really is split
        assert (b.labels[:bounds[1]] == c).any() and (b.labels[bounds[1]:] == c).any()
    check_sharded(b, bounds, 1, 1, 1e-10)
    check_sharded(b, bounds, 6, 3, 1e-9)


def test_rank_without_members_of_a_cluster():
    b = wl.make_random(300, 16, 3, K=3, mk_range=(2, 14), seed=211, dtype="f64")
    order = np.concatenate([np.nonzero(b.labels == 2)[0], np.nonzero(b.labels != 2)[0]])
    b = b.subset(order)                                       # cluster 2 first: rank 1 gets none of it
    n2 = int((b.labels == 2).sum())
    bounds = np.array([0, n2 + 40, b.N])
    assert not (b.labels[bounds[1]:] == 2).any() and (b.labels[bounds[1]:] == 0).any()
    check_sharded(b, bounds, 6, 3, 1e-9)


def test_rank_with_no_members():
    b = wl.make_random(200, 8, 2, K=2, mk_range=(1, 10), seed=212, dtype="f64")
    check_sharded(b, np.array([0, b.N, b.N]), 6, 3, 1e-9)


@pytest.mark.parametrize("fault", ["label", "weights"])
def test_rank_local_errors_agree(fault):
    b = wl.make_random(200, 8, 2, K=2, mk_range=(1, 10), seed=213, dtype="f64")
    res = run_ranks(b, shard_bounds(b.offsets, 2), 3, 3, faults={fault: 1}, timeout=300)
    assert res[0].get("error") == res[1].get("error") == 1          # AD2_ERR_ARG on both ranks


def test_fp32_config5_shape_two_ranks():
    """The bench workload's shape (d = 16, m = 32, Poisson supports) in fp32 with 2 ranks: same
    result as the unsharded run up to fp32 reordering, and the north_star full-schedule
    tolerances against the oracle."""
    b = wl.make_config(5, N=3000, K=6)
    bounds = shard_bounds(b.offsets, 2)
    one = run_ranks(b, np.array([0, b.N]), 20, 10)[0]
    two = run_ranks(b, bounds, 20, 10)
    np.testing.assert_array_equal(two[0]["w"], two[1]["w"])
    np.testing.assert_allclose(two[0]["w"], one["w"], atol=1e-6)
    ores, _ = oracle.run_bundle(b, T=20, tau=10, want_state=False)
    for c, r in ores.items():
        assert np.abs(two[0]["w"][c] - r.w).max() <= 1e-4
        assert_hybrid(two[0]["x"][c], r.x, 1e-3, floor=1.0, what=f"x c{c}")
