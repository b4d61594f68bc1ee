"""Seeded synthetic workloads for the B-ADMM barycenter path (shared by the oracle tests and the GPU path).

This module holds none of the centroid update's arithmetic (no cost matrix, no B-ADMM step,
no rho, no support update): it draws the ragged discrete distributions of BASELINE.json
``configs`` (recipes in SURVEY.md §8(d) and DESIGN.md "Input recipe") and the harness
initialisation that precedes the centroid update (k-means++ on member means, and a random
member merged down to m points by the paper's merge rule, §V P:820-840 Eq.merge).
That merge (``merge_to_size``) is the one piece of the paper's arithmetic here; it only produces
the initial centroids x0 / w0 that the oracle and the GPU path both read, never a compared
value (the oracle's own Eq.merge, ``oracle.merge``, and the device's ``ad2_merge_init`` are
tested against each other separately).  The paper's own datasets are not available;
these generators stand in for them (Table II is the shape model for
config 5).

Every stream is a ``numpy.random.Generator(PCG64)`` seeded from
``SeedSequence(seed, spawn_key=(config, purpose))`` so each purpose is independent and
reproducible.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

# purposes (spawn keys) — fixed forever, changing them changes every bundle
_P_SIZES, _P_COMP, _P_NOISE, _P_WEIGHTS, _P_CENTRES, _P_INIT, _P_SAMPLE, _P_PERM = range(8)


def _rng(seed: int, cfg: int, purpose: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(cfg, purpose))))


@dataclass
class Schedule:
    """Alg. 4 schedule: ``T`` iterations per round, support update every ``tau``."""
    T: int = 100
    tau: int = 10
    rounds: int = 1
    rho0: float = 2.0        # P:742 default
    eps: float = 1e-16       # P:588 ("e.g. 1e-16"); reading X3: same in fp32
    rule: int = 0            # 0 = R1 (Eq.badmmw), 1 = R2 (Eq.badmmw2)


@dataclass
class Bundle:
    """One shard-free instance: N ragged members, their labels, and K initial centroids.

    Layout follows the paper's problem statement: supports X = (x^(1)..x^(N)) as
    rows ``supports[offsets[k]:offsets[k+1]]`` (n x d, row-major), member weights w^(k) in
    ``weights`` (same slicing), labels l^(k) in [0, K), centroids x [K][m][d] and w [K][m].
    """
    name: str
    d: int
    m: int
    K: int
    offsets: np.ndarray      # int64 [N+1]
    supports: np.ndarray     # dtype [n, d]
    weights: np.ndarray      # dtype [n]
    labels: np.ndarray       # int32 [N]
    x0: np.ndarray           # dtype [K, m, d]
    w0: np.ndarray           # dtype [K, m]
    dtype: str = "f32"       # "f32" | "f64"
    sched: Schedule = field(default_factory=Schedule)

    @property
    def N(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def n(self) -> int:
        return int(self.offsets[-1])

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.offsets)

    def entries(self) -> int:
        """Plan entries per iteration, sum_k m * m_k (SURVEY.md §8 notation)."""
        return int(self.m * self.n)

    def member(self, k: int):
        a, b = int(self.offsets[k]), int(self.offsets[k + 1])
        return self.supports[a:b], self.weights[a:b]

    def subset(self, members: np.ndarray) -> "Bundle":
        """Bundle restricted to the given member indices (order kept)."""
        members = np.asarray(members, dtype=np.int64)
        sz = self.sizes[members]
        off = np.zeros(len(members) + 1, np.int64)
        np.cumsum(sz, out=off[1:])
        idx = _ragged_index(self.offsets[members], sz)
        return replace(self, offsets=off, supports=self.supports[idx], weights=self.weights[idx],
                       labels=self.labels[members])


def _ragged_index(starts: np.ndarray, sizes: np.ndarray) -> np.ndarray:
    tot = int(sizes.sum())
    if tot == 0:
        return np.zeros(0, np.int64)
    seg = np.repeat(np.arange(len(sizes)), sizes)
    off = np.zeros(len(sizes), np.int64)
    np.cumsum(sizes[:-1], out=off[1:])
    return starts[seg] + (np.arange(tot) - off[seg])


def _offsets(sizes: np.ndarray) -> np.ndarray:
    off = np.zeros(len(sizes) + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    return off


def _segment_normalise(v: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    s = np.add.reduceat(v, offsets[:-1])
    return v / np.repeat(s, np.diff(offsets))


_CHUNK = 1 << 22      # points per generator chunk (fixed: part of the workload definition)


def _chunk_rng(seed_rng_key, c: int):
    seed, cfg, purpose = seed_rng_key
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(cfg, purpose, c))))


def _parallel_chunks(n: int, fn):
    """Run fn(chunk_index, a, b) over fixed-size chunks on a thread pool (numpy's generators
    release the GIL); results depend only on the chunk index, not on the thread count."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    nch = (n + _CHUNK - 1) // _CHUNK
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda c: fn(c, c * _CHUNK, min(n, (c + 1) * _CHUNK)), range(nch)))


def _dirichlet_ragged(key, alpha: float, offsets: np.ndarray) -> np.ndarray:
    n = int(offsets[-1])
    g = np.empty(n, np.float64)

    def fill(c, a, b):
        g[a:b] = _chunk_rng(key, c).standard_gamma(alpha, size=b - a)
    _parallel_chunks(n, fill)
    # a member whose gammas all underflow would have no mass; gamma(alpha) never returns 0 in fp64
    return _segment_normalise(g, offsets)


def _zipf_ragged(rng, s: float, offsets: np.ndarray) -> np.ndarray:
    """w_j ∝ rank_j^-s over a random permutation of 1..m_k (SURVEY.md §8(d) cfg 4)."""
    sizes = np.diff(offsets)
    n = int(offsets[-1])
    seg = np.repeat(np.arange(len(sizes)), sizes)
    key = rng.random(n)
    order = np.lexsort((key, seg))              # random order inside each member
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n) - np.repeat(offsets[:-1], sizes)[order] + 1
    return _segment_normalise(rank.astype(np.float64) ** (-s), offsets)


def _gmm_points(key, means: np.ndarray, sigma: float, n: int, out_dtype) -> np.ndarray:
    """Each point picks a mixture component uniformly, plus N(0, sigma^2 I)."""
    ncomp, d = means.shape
    Y = np.empty((n, d), out_dtype)
    mt = means.astype(out_dtype)

    def fill(c, a, b):
        r = _chunk_rng(key, c)
        comp = r.integers(0, ncomp, size=b - a)
        noise = r.standard_normal((b - a, d), dtype=out_dtype)
        noise *= out_dtype(sigma)
        noise += mt[comp]
        Y[a:b] = noise
    _parallel_chunks(n, fill)
    return Y


def member_means(b: Bundle) -> np.ndarray:
    """Weighted mean of each member's support (harness feature for k-means++ init)."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    out = np.empty((b.N, b.d), np.float64)
    step = 1 << 18                                   # members per task

    def task(a):
        e = min(b.N, a + step)
        lo, hi = int(b.offsets[a]), int(b.offsets[e])
        Yw = b.supports[lo:hi].astype(np.float64) * b.weights[lo:hi].astype(np.float64)[:, None]
        out[a:e] = np.add.reduceat(Yw, b.offsets[a:e] - lo, axis=0)
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(task, range(0, b.N, step)))
    return out


def _nearest(points: np.ndarray, centres: np.ndarray, chunk: int = 1 << 16) -> np.ndarray:
    out = np.empty(len(points), np.int32)
    cc = (centres ** 2).sum(1)
    for a in range(0, len(points), chunk):
        p = points[a:a + chunk]
        dist = cc[None, :] - 2.0 * p @ centres.T          # + |p|^2, irrelevant for argmin
        out[a:a + chunk] = np.argmin(dist, axis=1)        # ties -> lowest index
    return out


def kmeanspp(points: np.ndarray, K: int, rng, lloyd_iters: int = 10) -> np.ndarray:
    """k-means++ D^2 seeding followed by Lloyd iterations (harness initialisation)."""
    n = len(points)
    centres = np.empty((K, points.shape[1]), np.float64)
    centres[0] = points[rng.integers(n)]
    d2 = ((points - centres[0]) ** 2).sum(1)
    for c in range(1, K):
        p = d2 / d2.sum() if d2.sum() > 0 else np.full(n, 1.0 / n)
        centres[c] = points[rng.choice(n, p=p)]
        d2 = np.minimum(d2, ((points - centres[c]) ** 2).sum(1))
    for _ in range(lloyd_iters):
        lab = _nearest(points, centres)
        cnt = np.bincount(lab, minlength=K)
        for t in range(points.shape[1]):
            s = np.bincount(lab, weights=points[:, t], minlength=K)
            centres[cnt > 0, t] = s[cnt > 0] / cnt[cnt > 0]
    return centres


def merge_to_size(x: np.ndarray, w: np.ndarray, m: int):
    """PAPER.md §V (Eq.merge): recursively merge the pair minimising
    w_i w_j |x_i-x_j|^2 / (w_i+w_j) into (w_i x_i + w_j x_j)/(w_i+w_j) until m points remain.
    If fewer than m points, duplicate the heaviest point with halved weights (SPEC.md fallback)."""
    x = [np.array(v, np.float64) for v in x]
    w = [float(v) for v in w]
    while len(w) > m:
        best, bi, bj = np.inf, 0, 1
        for i in range(len(w)):
            for j in range(i + 1, len(w)):
                c = w[i] * w[j] * float(((x[i] - x[j]) ** 2).sum()) / (w[i] + w[j])
                if c < best:
                    best, bi, bj = c, i, j
        wb = w[bi] + w[bj]
        xb = (w[bi] * x[bi] + w[bj] * x[bj]) / wb
        x[bi], w[bi] = xb, wb
        del x[bj], w[bj]
    while len(w) < m:
        h = int(np.argmax(w))
        w[h] *= 0.5
        x.append(x[h].copy())
        w.append(w[h])
    return np.array(x), np.array(w)


def init_centroids(b: Bundle, rng) -> tuple[np.ndarray, np.ndarray]:
    """Per cluster: a random member with m_k >= m (merged down to m if larger)."""
    x0 = np.zeros((b.K, b.m, b.d), np.float64)
    w0 = np.zeros((b.K, b.m), np.float64)
    sizes = b.sizes
    for c in range(b.K):
        mem = np.nonzero(b.labels == c)[0]
        if len(mem) == 0:
            raise ValueError(f"cluster {c} is empty")
        big = mem[sizes[mem] >= b.m]
        k = int(rng.choice(big)) if len(big) else int(mem[np.argmax(sizes[mem])])
        y, w = b.member(k)
        xx, ww = merge_to_size(y, w, b.m)
        x0[c], w0[c] = xx, ww / ww.sum()
    return x0, w0


def label_by_means(b: Bundle, K: int, rng_sample, rng_init, sample_frac: float = 0.1) -> np.ndarray:
    """k-means++ on the weighted member means of a sample, then every member -> nearest mean.
    Empty clusters are repaired by moving the member farthest from its mean (SPEC.md decision)."""
    mu = member_means(b)
    ns = max(K, int(round(sample_frac * b.N)))
    samp = rng_sample.choice(b.N, size=ns, replace=False)
    centres = kmeanspp(mu[samp], K, rng_init)
    lab = _nearest(mu, centres)
    counts = np.bincount(lab, minlength=K)
    while (counts == 0).any():
        c = int(np.nonzero(counts == 0)[0][0])
        dist = ((mu - centres[lab]) ** 2).sum(1)
        dist[counts[lab] <= 1] = -1.0
        k = int(np.argmax(dist))
        counts[lab[k]] -= 1
        lab[k] = c
        counts[c] += 1
        centres[c] = mu[k]
    return lab.astype(np.int32)


# ------------------------------------------------------------------------------------------
# BASELINE.json configs (1-based index as in SURVEY.md §8)
# ------------------------------------------------------------------------------------------

CONFIG_NAMES = {
    1: "cfg1_gmm2d_N200_m6_fp64",
    2: "cfg2_color3d_N20k_K10_m16",
    3: "cfg3_gmm16d_N200k_K64_m32",
    4: "cfg4_doc64d_N500k_K100_m64",
    5: "cfg5_gmm16d_N4M_K256_m32",
}

FULL_N = {1: 200, 2: 20_000, 3: 200_000, 4: 500_000, 5: 4_000_000}


def make_config(cfg: int, N: Optional[int] = None, K: Optional[int] = None, seed: int = 0,
                dtype: Optional[str] = None) -> Bundle:
    """Build config ``cfg`` (1..5) at its full size, or with N (and K) overridden for small parity cases."""
    N = FULL_N[cfg] if N is None else int(N)
    ck = cfg  # spawn-key namespace
    rs = lambda p: _rng(seed, ck, p)
    if cfg == 1:
        d, m, Kc = 2, 6, 1
        sizes = np.full(N, 6, np.int64)
        off = _offsets(sizes)
        means = rs(_P_CENTRES).uniform(-5.0, 5.0, size=(3, d))
        Y = _gmm_points((seed, ck, _P_NOISE), means, 1.0, int(off[-1]), np.float64)
        W = _dirichlet_ragged((seed, ck, _P_WEIGHTS), 1.0, off)
        labels = np.zeros(N, np.int32)
        pick = rs(_P_INIT).choice(int(off[-1]), size=m, replace=False)   # X9: 6 distinct pooled points
        x0 = Y[pick][None].astype(np.float64)
        w0 = np.full((1, m), 1.0 / m)
        sched = Schedule(T=100, tau=20)
        b = Bundle(CONFIG_NAMES[1], d, m, Kc, off, Y, W, labels, x0, w0, dtype or "f64", sched)
        return _cast(b)
    if cfg == 2:
        d, m, Kc = 3, 16, 10
        sizes = rs(_P_SIZES).integers(8, 17, size=N).astype(np.int64)
        off = _offsets(sizes)
        centres = rs(_P_CENTRES).uniform(0.0, 1.0, size=(32, d))
        Y = _gmm_points((seed, ck, _P_NOISE), centres, 0.05, int(off[-1]), np.float64)
        W = _dirichlet_ragged((seed, ck, _P_WEIGHTS), 1.0, off)
        sched = Schedule(T=100, tau=10, rounds=10)
    elif cfg in (3, 5):
        d, m, Kc = 16, 32, (64 if cfg == 3 else 256)
        sizes = np.clip(rs(_P_SIZES).poisson(20.0, size=N), 4, 32).astype(np.int64)
        off = _offsets(sizes)
        means = 2.0 * rs(_P_CENTRES).standard_normal((64, d))            # N(0, 4 I)
        Y = _gmm_points((seed, ck, _P_NOISE), means, 1.0, int(off[-1]), np.float32)
        W = _dirichlet_ragged((seed, ck, _P_WEIGHTS), 0.5, off)
        sched = Schedule(T=50, tau=10, rounds=10 if cfg == 3 else 3)
    elif cfg == 4:
        d, m, Kc = 64, 64, 100
        sizes = rs(_P_SIZES).integers(20, 65, size=N).astype(np.int64)
        off = _offsets(sizes)
        topics = rs(_P_CENTRES).standard_normal((1000, d))
        topics /= np.linalg.norm(topics, axis=1, keepdims=True)
        n = int(off[-1])
        doc_topic = rs(_P_COMP).integers(0, 1000, size=N)
        pt_topic = np.repeat(doc_topic, sizes)
        Y = np.empty((n, d), np.float32)
        rn = rs(_P_NOISE)
        ch = 1 << 21
        for a in range(0, n, ch):
            bb = min(n, a + ch)
            v = topics[pt_topic[a:bb]] + 0.3 * rn.standard_normal((bb - a, d)) / 8.0   # g ~ N(0, I/64)
            Y[a:bb] = v / np.linalg.norm(v, axis=1, keepdims=True)
        W = _zipf_ragged(rs(_P_WEIGHTS), 1.1, off)
        sched = Schedule(T=50, tau=10, rounds=5)
    else:
        raise ValueError(cfg)
    if K is not None:
        Kc = int(K)
    tmp = Bundle(CONFIG_NAMES[cfg], d, m, Kc, off, Y, W, np.zeros(N, np.int32),
                 np.zeros((Kc, m, d)), np.zeros((Kc, m)), dtype or "f32", sched)
    tmp.labels = label_by_means(tmp, Kc, rs(_P_SAMPLE), rs(_P_INIT))
    tmp.x0, tmp.w0 = init_centroids(tmp, rs(_P_PERM))
    if N != FULL_N[cfg] or K is not None:
        tmp.name = f"{CONFIG_NAMES[cfg]}@N{N}K{Kc}"
    return _cast(tmp)


def _cast(b: Bundle) -> Bundle:
    """Store floats in the bundle dtype; weights are renormalised in fp64 before the cast."""
    ft = np.float64 if b.dtype == "f64" else np.float32
    b.supports = np.ascontiguousarray(b.supports, dtype=ft)
    b.weights = np.ascontiguousarray(b.weights, dtype=ft)
    b.x0 = np.ascontiguousarray(b.x0, dtype=ft)
    b.w0 = np.ascontiguousarray(b.w0 / b.w0.sum(1, keepdims=True), dtype=ft)
    b.offsets = np.ascontiguousarray(b.offsets, dtype=np.int64)
    b.labels = np.ascontiguousarray(b.labels, dtype=np.int32)
    return b


def make_random(N: int, m: int, d: int, K: int = 1, mk_range=(1, 8), seed: int = 0, dtype: str = "f64",
                alpha: float = 1.0, T: int = 10, tau: int = 5, rule: int = 0, spread: float = 1.0) -> Bundle:
    """Small generic instance (for pins, ragged edge cases and parity at odd shapes)."""
    ck = 100
    rs = lambda p: _rng(seed, ck, p)
    lo, hi = mk_range
    sizes = rs(_P_SIZES).integers(lo, hi + 1, size=N).astype(np.int64)
    off = _offsets(sizes)
    Y = spread * rs(_P_NOISE).standard_normal((int(off[-1]), d))
    W = _dirichlet_ragged((seed, ck, _P_WEIGHTS), alpha, off)
    labels = (np.arange(N) % K).astype(np.int32)
    rs(_P_SAMPLE).shuffle(labels)
    x0 = spread * rs(_P_INIT).standard_normal((K, m, d))
    w0 = _dirichlet_ragged((seed, ck, _P_CENTRES), 2.0, _offsets(np.full(K, m))).reshape(K, m)
    b = Bundle(f"random_N{N}_m{m}_d{d}_K{K}", d, m, K, off, Y, W, labels, x0, w0, dtype,
               Schedule(T=T, tau=tau, rule=rule))
    return _cast(b)


@dataclass
class SymbolicBundle:
    """Members over a fixed symbol set with a symbol-to-symbol cost table."""
    name: str
    V: int
    m: int
    K: int
    D: np.ndarray            # [V][V] cost table
    offsets: np.ndarray      # [N+1]
    ids: np.ndarray          # [n] int32 symbol ids
    weights: np.ndarray      # [n]
    labels: np.ndarray       # [N] int32
    xs0: np.ndarray          # [K][m] int32 centroid symbols
    w0: np.ndarray           # [K][m]
    dtype: str = "f32"
    sched: Schedule = field(default_factory=lambda: Schedule(T=30, tau=10))

    @property
    def N(self) -> int:
        return len(self.offsets) - 1


def make_symbolic(N: int = 600, K: int = 5, m: int = 16, V: int = 400, mk_range=(5, 40), seed: int = 0,
                  dtype: str = "f32") -> SymbolicBundle:
    """Seeded stand-in for the paper's symbolic data (protein n-gram histograms, P:892-893,
    dataset missing): V = 400 symbols (dipeptide-like), each with a random 6-D profile; the cost
    table is the L1 distance between profiles (non-Euclidean, non-negative).  K latent groups
    each prefer a random 60-symbol subset (Zipf over it, 20 % background); a member draws
    m_k ~ U{mk_range} distinct symbols from its group's law, weights Dirichlet(1).  Labels are
    random; each centroid starts from m distinct symbols of its first member's group law."""
    ck = 200
    rs = lambda p: _rng(seed, ck, p)
    prof = rs(_P_CENTRES).uniform(0.0, 1.0, size=(V, 6))
    D = np.abs(prof[:, None, :] - prof[None, :, :]).sum(-1)
    g = rs(_P_COMP)
    laws = []
    for _ in range(K):
        fav = g.choice(V, 60, replace=False)
        p = np.full(V, 0.2 / V)
        p[fav] += 0.8 * (1.0 / np.arange(1, 61)) / (1.0 / np.arange(1, 61)).sum()
        laws.append(p / p.sum())
    lo, hi = mk_range
    sizes = rs(_P_SIZES).integers(lo, hi + 1, size=N).astype(np.int64)
    off = _offsets(sizes)
    grp = rs(_P_SAMPLE).integers(0, K, size=N)
    rn = rs(_P_NOISE)
    ids = np.concatenate([rn.choice(V, int(sizes[k]), replace=False, p=laws[grp[k]]) for k in range(N)])
    W = _dirichlet_ragged((seed, ck, _P_WEIGHTS), 1.0, off)
    labels = rs(_P_PERM).integers(0, K, size=N).astype(np.int32)
    for c in range(K):                                   # no empty cluster
        labels[c % N] = c
    xs0 = np.stack([rs(_P_INIT).choice(V, m, replace=False, p=laws[grp[int(np.nonzero(labels == c)[0][0])]])
                    for c in range(K)]).astype(np.int32)
    w0 = np.full((K, m), 1.0 / m)
    ft = np.float64 if dtype == "f64" else np.float32
    return SymbolicBundle(f"symbolic_V{V}_N{N}_K{K}_m{m}", V, m, K, np.ascontiguousarray(D, ft),
                          np.ascontiguousarray(off, np.int64), np.ascontiguousarray(ids, np.int32),
                          np.ascontiguousarray(W, ft), labels, xs0, np.ascontiguousarray(w0, ft), dtype)
