"""fp64 CPU ORACLE for the initial partition of AD2-clustering.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module; the product package never
imports it and shares no code with it.

Alg. 1 starts from "K random centroid[s]" and a labelling; the paper does not fix how.
SURVEY.md §8(d) fixes the recipe (SURVEY.md:557): k-means++ D^2 seeding and Lloyd iterations on
the weighted member means of a sample (the paper's own comparison method, "Kmeans++"),
every member labelled to its nearest mean, then per cluster a random member with at least m
support points whose support Eq.merge reduces to m points (``oracle.merge``).

Every random draw is an INPUT (sample indices, uniforms u in [0, 1)), so the oracle and the CUDA
path see the same draws; the readings that turn a draw into an index are DESIGN.md X20-X23:
  X20  first centre: sample point floor(u_0 * ns); centre c > 0: the first sample index i whose
       inclusive prefix sum of D^2 exceeds u_c * (sum of D^2) (inverse-CDF sampling of
       P(i) = D_i^2 / sum D^2); if every D^2 is 0, sample point floor(u_c * ns).
  X21  squared distances are sum_t (p_t - c_t)^2 accumulated in coordinate order t = 0..d-1
       (multiply and add rounded separately); nearest centre: ties to the lowest index;
       a Lloyd centre is the mean of its points summed in index order (an empty cluster keeps
       its centre).
  X22  empty clusters after labelling all members: the lowest empty cluster takes the member
       farthest from its own centre among clusters with >= 2 members (lowest index on ties) and
       that member's mean becomes its centre; repeat.
  X23  the picked member of cluster c: among c's members with m_k >= m in index order, the one at
       position floor(u_c * n_big); if there is none, the first member of c with the largest m_k.
Plain numpy, vectorised over points only; every sum has the order stated above.
"""
from __future__ import annotations

import numpy as np


def member_means(offsets, Y, omega) -> np.ndarray:
    """mean(P^(k)) = sum_j w_j^(k) y_j (P^(k) = {(w_j, y_j)}; weights on the simplex),
    accumulated over j in order; fp32 inputs are widened to fp64 first."""
    off = np.asarray(offsets, np.int64)
    Y = np.asarray(Y, np.float64)
    om = np.asarray(omega, np.float64)
    N, d = len(off) - 1, Y.shape[1]
    mk = np.diff(off)
    mu = np.zeros((N, d))
    for j in range(int(mk.max()) if N else 0):
        has = mk > j
        idx = off[:-1][has] + j
        mu[has] = mu[has] + om[idx, None] * Y[idx]
    return mu


def sq_dist(P: np.ndarray, c: np.ndarray) -> np.ndarray:
    """|p - c|^2 for every row p of P (X21: coordinate order, no fused multiply-add)."""
    acc = np.zeros(len(P))
    for t in range(P.shape[1]):
        diff = P[:, t] - c[t]
        acc = acc + diff * diff
    return acc


def nearest(P: np.ndarray, centres: np.ndarray) -> np.ndarray:
    """argmin_c |p - centre_c|^2, ties to the lowest c (X21)."""
    D = np.stack([sq_dist(P, c) for c in centres], axis=1)
    return np.argmin(D, axis=1).astype(np.int32)


def kmeanspp(P, K: int, u, lloyd_iters: int) -> np.ndarray:
    """k-means++ D^2 seeding (X20) followed by lloyd_iters Lloyd iterations (X21) on the points
    P [ns][d]; u [K] uniforms in [0, 1).  Returns the centres [K][d]."""
    P = np.asarray(P, np.float64)
    u = np.asarray(u, np.float64)
    ns = len(P)
    centres = np.empty((K, P.shape[1]))
    centres[0] = P[min(int(u[0] * ns), ns - 1)]
    d2 = sq_dist(P, centres[0])
    for c in range(1, K):
        cum = np.cumsum(d2)                           # inclusive prefix, index order
        total = cum[-1]
        if total > 0:
            i = int(np.searchsorted(cum, u[c] * total, side="right"))
            if i >= ns:                               # u*total rounded up to total: last positive D^2
                i = int(np.nonzero(d2 > 0)[0][-1])
        else:
            i = min(int(u[c] * ns), ns - 1)
        centres[c] = P[i]
        d2 = np.minimum(d2, sq_dist(P, centres[c]))
    for _ in range(lloyd_iters):
        lab = nearest(P, centres)
        cnt = np.bincount(lab, minlength=K)
        for t in range(P.shape[1]):
            s = np.bincount(lab, weights=P[:, t], minlength=K)     # index order per cluster
            centres[cnt > 0, t] = s[cnt > 0] / cnt[cnt > 0]
    return centres


def label_nearest(mu, centres):
    """Every member to its nearest centre (X21), then the empty-cluster repair (X22).
    Returns (labels int32 [N], centres [K][d] after the repair)."""
    mu = np.asarray(mu, np.float64)
    centres = np.array(centres, np.float64)
    K = len(centres)
    if len(mu) < K:
        raise ValueError("label_nearest needs N >= K (X22: a donor cluster with >= 2 members)")
    lab = nearest(mu, centres)
    counts = np.bincount(lab, minlength=K)
    while (counts == 0).any():
        c = int(np.nonzero(counts == 0)[0][0])
        dist = np.empty(len(mu))
        for e in range(K):                            # each member against its own centre
            sel = lab == e
            dist[sel] = sq_dist(mu[sel], centres[e])
        dist[counts[lab] <= 1] = -1.0
        k = int(np.argmax(dist))                      # first maximum
        counts[lab[k]] -= 1
        lab[k] = c
        counts[c] += 1
        centres[c] = mu[k]
    return lab, centres


def seed_labels(offsets, Y, omega, sample, K: int, u, lloyd_iters: int):
    """The whole initial partition: member means -> k-means++ on the sampled means -> labels.
    Returns (labels int32 [N], centres [K][d] after the repair)."""
    mu = member_means(offsets, Y, omega)
    centres = kmeanspp(mu[np.asarray(sample, np.int64)], K, u, lloyd_iters)
    return label_nearest(mu, centres)


def pick_members(offsets, labels, m: int, u) -> np.ndarray:
    """X23: per cluster the member whose support initialises the centroid."""
    mk = np.diff(np.asarray(offsets, np.int64))
    labels = np.asarray(labels)
    K = len(u)
    pick = np.full(K, -1, np.int64)
    for c in range(K):
        mem = np.nonzero(labels == c)[0]
        if len(mem) == 0:
            continue
        big = mem[mk[mem] >= m]
        if len(big):
            pick[c] = big[min(int(u[c] * len(big)), len(big) - 1)]
        else:
            pick[c] = mem[int(np.argmax(mk[mem]))]
    return pick
