"""Time the GPU assignment step (ad2_assign) on a BASELINE config after one B-ADMM round
(diagnostic for DESIGN.md / profiles; not a bench number)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--N", type=int, default=None)
args = ap.parse_args()
b = wl.make_config(args.cfg, N=args.N)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = [dev(a) for a in (b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0)]
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)
s = b.sched
ctx.init(*D, b.K, b.m, s.rho0, s.eps, s.rule, dtype=b.dtype)
ad2.run_schedule(ctx, s.T, s.tau)
x, w = ctx.centroids()
xd, wd = dev(x), dev(w)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    lab, w2, n_exact = ctx.assign(D[0], D[1], D[2], xd, wd, dtype=b.dtype)
    dt = time.perf_counter() - t
    changed = float(np.mean(lab != b.labels))
    print(f"{b.name}: assign {1e3 * dt:.1f} ms, N={b.N} K={b.K}, exact solves {n_exact} "
          f"({n_exact / b.N:.2f}/member, {n_exact / (b.N * b.K):.3f} of all pairs), labels changed {changed:.3f}",
          flush=True)
