"""One B-ADMM round on a BASELINE config through the C ABI (used under ncu for launch lists
and kernel captures; never a bench number)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--N", type=int, default=None)
ap.add_argument("--rounds", type=int, default=1)
ap.add_argument("--state-mode", type=int, default=0)
ap.add_argument("--tc", type=int, default=-1, help="ad2_set_tc_cost (1/0); -1: library default")
ap.add_argument("--cost-mode", type=int, default=0, help="params cost_mode (1: bf16 tensor-core cost build)")
args = ap.parse_args()
b = wl.make_config(args.cfg, N=args.N)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = [dev(a) for a in (b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0)]
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.set_state_mode(args.state_mode)
if args.tc >= 0:
    ctx.set_tc_cost(args.tc)
s = b.sched
for r in range(args.rounds):
    ctx.init(*D, b.K, b.m, s.rho0, s.eps, s.rule, dtype=b.dtype, cost_mode=args.cost_mode)
    ad2.run_schedule(ctx, s.T, s.tau)
    obj = ctx.objective()
torch.cuda.synchronize()
print("ok", b.name, ctx.info(), float(obj.mean()))
