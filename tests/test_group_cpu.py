"""The host process group (ad2_group_*, include/ad2.h) on CPU, world size 2 and 3: libad2's
transport for the per-cluster partial sums when ranks are processes on one host.
It is host code, so it runs here without a GPU.  Checked: the sum of every rank's buffer, in
every dtype, bit-identical on all ranks and equal to the rank-order sum; several consecutive
collectives (barrier reuse); a missing peer times out instead of hanging."""
import multiprocessing as mp
import os
import uuid

import numpy as np
import pytest


def _rank(name, world, rank, q):
    try:
        from paper_1510_00012_b200 import ad2
        g = ad2.Group(name, world, rank, slot_bytes=1 << 16)
        out = []
        for it in range(20):
            rng = np.random.default_rng(1000 * it + rank)
            a = rng.standard_normal(1000).astype(np.float32)
            b = rng.standard_normal(37)
            c = rng.integers(0, 1 << 40, 5).astype(np.uint64)
            g.allreduce(a)
            g.allreduce(b)
            g.allreduce(c)
            out.append((a.copy(), b.copy(), c.copy()))
        g.close()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_group_allreduce_rank_order_sum(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/ad2t_{uuid.uuid4().hex[:12]}"
    ps = [ctx.Process(target=_rank, args=(name, world, r, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(30)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    for it in range(20):
        want = []
        for dt, n, j in ((np.float32, 1000, 0), (np.float64, 37, 1), (np.uint64, 5, 2)):
            parts = []
            for r in range(world):
                rng = np.random.default_rng(1000 * it + r)
                a = rng.standard_normal(1000).astype(np.float32)
                b = rng.standard_normal(37)
                c = rng.integers(0, 1 << 40, 5).astype(np.uint64)
                parts.append((a, b, c)[j])
            s = parts[0].copy()
            for p_ in parts[1:]:
                s = (s + p_).astype(dt)                       # rank order 0, 1, ... in the dtype
            want.append(s)
        for r in range(world):
            for j in range(3):
                np.testing.assert_array_equal(res[r][it][j], want[j])


def test_group_missing_peer_times_out():
    from paper_1510_00012_b200 import ad2
    os.environ["AD2_GROUP_TIMEOUT"] = "1"
    try:
        with pytest.raises(ad2.AD2Error, match="STATE"):
            ad2.Group(f"/ad2t_{uuid.uuid4().hex[:12]}", 2, 0)
    finally:
        del os.environ["AD2_GROUP_TIMEOUT"]


def test_group_rejects_bad_arguments():
    from paper_1510_00012_b200 import ad2
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ad2.Group("no_leading_slash", 2, 0)
    with pytest.raises(ad2.AD2Error, match="ARG"):
        ad2.Group("/x", 2, 2)
    g = ad2.Group(f"/ad2t_{uuid.uuid4().hex[:12]}", 1, 0, slot_bytes=64)
    a = np.arange(4.0)
    np.testing.assert_array_equal(g.allreduce(a), np.arange(4.0))        # one rank: identity
    with pytest.raises(ad2.AD2Error):
        g.allreduce(np.zeros(100))                                       # larger than the slot
    g.close()
