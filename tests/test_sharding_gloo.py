"""Multi-rank host logic on CPU (gloo, world size 2): entry-balanced shard bounds, the NCCL-id
bootstrap, and the decomposition the multi-GPU path relies on — every cross-member quantity of
Alg. 4 (rho numerator and counts, the w consensus sums, the x-update sums, the objective) is a
sum over shards of per-member terms, so all-reducing per-shard partial sums reproduces the
unsharded run.  The per-member terms come from the fp64 oracle's single-formula functions."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1510_00012_b200 import workloads as wl
from paper_1510_00012_b200.sharding import shard_bounds, bootstrap_nccl


def test_shard_bounds_cover_and_balance():
    b = wl.make_config(3, N=5000, K=8)
    for world in (1, 2, 3, 4, 8):
        bd = shard_bounds(b.offsets, world)
        assert bd[0] == 0 and bd[-1] == b.N and (np.diff(bd) >= 0).all()
        pts = np.diff(b.offsets[bd])
        assert pts.max() - pts.min() <= 2 * b.sizes.max() + 1          # balanced by plan entries
    assert list(shard_bounds(np.array([0, 5, 6, 7, 8]), 2)) == [0, 1, 4]


def test_shard_bounds_degenerate():
    assert list(shard_bounds(np.array([0]), 3)) == [0, 0, 0, 0]        # no members at all
    bd = shard_bounds(np.array([0, 3]), 4)                              # one member, 4 ranks
    assert bd[0] == 0 and bd[-1] == 1 and (np.diff(bd) >= 0).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_alg4(rank, world, port, T, tau, rule, q):
    """Alg. 4 on this rank's shard with gloo all-reduce of per-cluster partial sums (the same
    decomposition libad2 uses with NCCL)."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = wl.make_random(60, 4, 2, K=1, mk_range=(1, 6), seed=31, dtype="f64")
        bd = shard_bounds(b.offsets, world)
        mine = range(bd[rank], bd[rank + 1])
        x, w = b.x0[0].copy(), b.w0[0].copy()
        m = b.m

        def allsum(v):
            t = torch.tensor(np.asarray(v, np.float64))
            dist.all_reduce(t)
            return t.numpy()

        Y = {k: b.member(k)[0].astype(np.float64) for k in mine}
        om = {k: b.member(k)[1] / b.member(k)[1].sum() for k in mine}
        C = {k: oracle.cost(x, Y[k]) for k in mine}
        s = allsum([sum(C[k].sum() for k in mine), sum(m * len(om[k]) for k in mine)])
        rho = 2.0 * s[0] / s[1]
        P2 = {k: np.outer(w, om[k]) for k in mine}
        L = {k: np.zeros_like(P2[k]) for k in mine}
        for t in range(1, T + 1):
            P1, B, R = {}, {}, {}
            part = np.zeros(m)
            for k in mine:
                P1[k] = oracle.pi1(P2[k], L[k], C[k], om[k], rho)
                B[k] = oracle.pi1_tilde(P1[k], L[k], rho)
                R[k], wt = oracle.rowmass(B[k])
                part += np.sqrt(wt) if rule == 1 else wt
            S = allsum(part)
            w = S * S if rule == 1 else S
            w = w / w.sum()
            for k in mine:
                P2[k] = oracle.pi2(B[k], w)
                L[k] = oracle.dual(L[k], P1[k], P2[k], rho)
            if t % tau == 0:
                num = np.zeros((m, b.d + 1))
                for k in mine:
                    num[:, :b.d] += P2[k] @ Y[k]
                    num[:, b.d] += P2[k].sum(1)
                num = allsum(num)
                keep = w < 1e-12
                x = np.where(keep[:, None], x, num[:, :b.d] / num[:, b.d:])
                C = {k: oracle.cost(x, Y[k]) for k in mine}
        obj = allsum([sum((C[k] * P1[k]).sum() for k in mine)])[0] / b.N
        if rank == 0:
            q.put((x, w, rho, obj))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rule", [0, 1])
def test_sharded_allreduce_equals_unsharded_oracle(rule):
    T, tau, world = 12, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_alg4, args=(r, world, port, T, tau, rule, q)) for r in range(world)]
    for p in procs:
        p.start()
    x, w, rho, obj = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    b = wl.make_random(60, 4, 2, K=1, mk_range=(1, 6), seed=31, dtype="f64")
    r = oracle.badmm_centroid(b.x0[0], b.w0[0], b.offsets, b.supports, b.weights, T, tau, rule)
    assert rho == pytest.approx(r.rho, rel=1e-13)
    np.testing.assert_allclose(w, r.w, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(x, r.x, rtol=1e-11, atol=1e-12)
    assert obj == pytest.approx(r.obj, rel=1e-11)


def _bootstrap(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_00012_b200 import ad2
        ad2.nccl_unique_id = lambda: bytes(range(128))     # no GPU / NCCL on this host

        class FakeCtx:
            def attach_nccl(self, n, r, uid):
                q.put((r, n, uid))
        bootstrap_nccl(FakeCtx())
    finally:
        dist.destroy_process_group()


def test_bootstrap_broadcasts_rank0_unique_id():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bootstrap, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=60), q.get(timeout=60)])
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    assert got[0][:2] == (0, 2) and got[1][:2] == (1, 2)
    assert got[0][2] == got[1][2] == bytes(range(128))
