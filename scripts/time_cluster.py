"""The AD2 outer loop (ad2_cluster) on a BASELINE config: rounds, label changes and wall time
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
ap.add_argument("--rounds", type=int, default=10)
ap.add_argument("--stop", type=float, default=0.001)
args = ap.parse_args()
b = wl.make_config(args.cfg, N=args.N)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = [dev(a) for a in (b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0)]
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)
s = b.sched
torch.cuda.synchronize()
t = time.perf_counter()
res = ctx.cluster(*D, b.K, b.m, s.T, s.tau, args.rounds, stop_frac=args.stop, dtype=b.dtype)
torch.cuda.synchronize()
dt = time.perf_counter() - t
obj = res["objective"]
print(f"{b.name}: {res['rounds']} rounds in {dt:.2f} s ({dt / res['rounds']:.3f} s/round incl. assignment)")
print("changed fraction per round:", np.round(res["changed"], 4).tolist())
print("mean surrogate objective per round:", np.round(obj.mean(1), 4).tolist())
