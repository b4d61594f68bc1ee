"""Diagnostic: where the compressed state (mode 1) departs from the oracle most, config 5 shape."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1510_00012_b200 import ad2, workloads as wl
from tests.harness import run_gpu

b = wl.make_config(5, N=3000)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
res = {}
for mode in (0, 1):
    ctx, rho, _ = run_gpu(b, T, T, state_mode=mode)
    res[mode] = (ctx.centroids(), ctx.member_matrices(ad2.PI2), ctx.member_matrices(ad2.PI1), rho)
ores, members = oracle.run_bundle(b, T=T, tau=T)
for mode in (0, 1):
    (x, w), P2, P1, rho = res[mode]
    worst = (0, None)
    for c, r in ores.items():
        for k, M in zip(members[c], r.mats["Pi2"]):
            G = P2[k].astype(np.float64)
            mx = max(abs(M).max(), 1e-300)
            allmax = max(abs(MM).max() for MM in r.mats["Pi2"])
            err = np.abs(G - M) / (np.abs(M) + 1e-4 * allmax)
            i, j = np.unravel_index(np.argmax(err), err.shape)
            if err[i, j] > worst[0]:
                y, om = b.member(k)
                C = ((b.x0[c].astype(np.float64)[:, None, :] - y[None].astype(np.float64)) ** 2).sum(-1)
                worst = (err[i, j], dict(c=c, k=int(k), i=int(i), j=int(j), got=G[i, j], want=M[i, j],
                                         col=M[:, j], C_rho=C[:, j] / r.rho, om=float(om[j]), w_i=r.w[i],
                                         Cij_rho=C[i, j] / r.rho, mk=len(om)))
    e, info = worst
    print(f"mode {mode}: worst hybrid {e:.3g}")
    for kk, v in info.items():
        if kk in ("col", "C_rho"):
            print("   ", kk, np.array2string(np.asarray(v), precision=3, max_line_width=200))
        else:
            print("   ", kk, v)
for mode in (0, 1):
    (x, w), P2, P1, rho = res[mode]
    errs = []
    for c, r in ores.items():
        d = np.abs(x[c].astype(np.float64) - r.x)
        i = np.unravel_index(np.argmax(d), d.shape)
        errs.append((d.max() / np.abs(r.x).max(), c, i, r.w[i[0]], float(w[c][i[0]])))
    errs.sort(reverse=True)
    print(f"mode {mode} x worst:", errs[:3])
