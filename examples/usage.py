"""The README's usage example, runnable: one centroid update, the assignment step, the AD2 loop
and the initial partition (k-means++, nearest labels, member picks, Eq.merge) on a small seeded config-3 workload (needs a B200)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402

b = wl.make_config(3, N=20_000, K=16)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)

rho = ctx.init(dev(b.offsets), dev(b.supports), dev(b.weights), dev(b.labels), dev(b.x0), dev(b.w0),
               b.K, b.m, rho0=2.0, eps=1e-16, rule=ad2.R1)
ad2.run_schedule(ctx, T=50, tau=10)
obj = ctx.objective()
x, w = ctx.centroids()
print("rho[:3]", rho[:3], "objective[:3]", obj[:3])

labels, w2, n_exact = ctx.assign(dev(b.offsets), dev(b.supports), dev(b.weights), dev(x), dev(w))
print("labels changed by one assignment:", float(np.mean(labels != b.labels)), "exact solves:", n_exact)

res = ctx.cluster(dev(b.offsets), dev(b.supports), dev(b.weights), dev(b.labels), dev(b.x0), dev(b.w0),
                  b.K, b.m, T=50, tau=10, max_rounds=4, stop_frac=0.001)
print("loop:", res["rounds"], "rounds, changed", np.round(res["changed"], 4))

rng = np.random.default_rng(0)
cen = ctx.kmeanspp(dev(b.offsets), dev(b.supports), dev(b.weights), rng.choice(b.N, 2000, replace=False),
                   rng.uniform(size=b.K), 10)
labels0, cen = ctx.label_nearest(dev(b.offsets), dev(b.supports), dev(b.weights), cen)
print("initial partition: cluster sizes", np.bincount(labels0, minlength=b.K).min(), "..",
      np.bincount(labels0, minlength=b.K).max())
pick = ctx.pick_members(dev(b.offsets), dev(b.supports), dev(b.weights), dev(labels0), b.m, rng.uniform(size=b.K))
x0, w0 = ctx.merge_init(dev(b.offsets), dev(b.supports), dev(b.weights), pick, b.K, b.m)
print("merge init:", x0.shape, float(w0.sum(1).min()), float(w0.sum(1).max()))
