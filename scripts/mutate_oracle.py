#!/usr/bin/env python
"""Mutation test of the oracle's pins: apply one plausible mistake at a time to a scratch copy of
oracle/*.c and check that `tests/test_oracle_pins.py` (the -m "not gpu" pins) FAILS.

    python scripts/mutate_oracle.py            # all mutations, table on stdout
    python scripts/mutate_oracle.py M6 M13     # a subset

A mutation that survives every pin is a hole in the oracle's pinning (DESIGN.md §3 lists the
table).  Equivalent mutations (identical results up to rounding) are not listed.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC = "oracle/ad2_oracle.c"
OT = "oracle/ad2_oracle_ot.c"
SEED = "oracle/seed.py"

# id: (file, old, new, occurrence (1-based), what it models)
MUTATIONS = {
    "M1": (ORC, "exp((C[i * mk + j] + Lam[i * mk + j]) / (-rho))", "exp((C[i * mk + j] + Lam[i * mk + j]) / (rho))", 1,
           "Eq.badmmc0b exp sign"),
    "M2": (ORC, "for (int l = 0; l < m; ++l) colsum += pt[l * mk + j];",
           "for (int l = 0; l < m; ++l) colsum += pt[l * mk + (j + 1) % mk];", 1, "Eq.badmmc0 column index"),
    "M3": (ORC, "ad2o_update_support(m, d, x, w, N, off, Y, Pi2);", "ad2o_update_support(m, d, x, w, N, off, Y, Pi1);", 1,
           "X5: Eq.updatex fed Pi1 instead of Pi2"),
    "M4": (ORC, "ad2o_pi1_tilde(m, mk, Pi1 + b, Lam + b, rho, eps, B + b);",
           "ad2o_dual(m, mk, Lam + b, Pi1 + b, Pi2 + b, rho); ad2o_pi1_tilde(m, mk, Pi1 + b, Lam + b, rho, eps, B + b);"
           " ad2o_dual(m, mk, Lam + b, Pi2 + b, Pi1 + b, rho);", 1,
           "X4: Eq.badmmc1b with Lambda after a dual step on the old Pi2"),
    "M5": (ORC, "double rho = rho0 * sumC / ((double)m * (double)n);",
           "double rho = rho0 * sumC / ((double)m * (double)n * (double)N);", 1, "X1: in-loop rho with the extra 1/N"),
    "M6": (ORC, "Pi2[i * mk + j] * exp((C[i * mk + j] + Lam[i * mk + j]) / (-rho)) + eps;",
           "Pi2[i * mk + j] * (exp((C[i * mk + j] + Lam[i * mk + j]) / (-rho)) + eps);", 1,
           "X3: eps inside the product in Eq.badmmc0b"),
    "M7": (ORC, "*obj_out = (T > 0) ? ad2o_surrogate(m, d, x, N, off, Y, Pi1) : NAN;",
           "*obj_out = (T > 0) ? ad2o_surrogate(m, d, x, N, off, Y, Pi2) : NAN;", 1, "X14: objective with Pi2"),
    "M8": (ORC, "rho * (Pi1[i * mk + j] - Pi2[i * mk + j])", "rho * (Pi2[i * mk + j] - Pi1[i * mk + j])", 1,
           "Eq.badmm2 sign"),
    "M9": (ORC, "w[i] = (rule == 1) ? s * s : s;", "w[i] = s;", 1, "Eq.badmmw2 without the square"),
    "M10": (ORC, "Pi2[i * mk + j] = B[i * mk + j] / rowsum * w[i];", "Pi2[i * mk + j] = B[i * mk + j] * w[i];", 1,
            "Eq.badmmc1 without the row normalisation"),
    "M11": (ORC, "if (w[i] < 1e-12) continue;", "", 1, "X12 guard dropped"),
    "M13": (ORC, "B[i * mk + j] = Pi1[i * mk + j] * exp(Lam[i * mk + j] / rho) + eps;",
            "B[i * mk + j] = Pi1[i * mk + j] * exp(Lam[i * mk + j] / rho);", 1, "X3: eps dropped in Eq.badmmc1b"),
    "M14": (ORC, "B[i * mk + j] = Pi1[i * mk + j] * exp(Lam[i * mk + j] / rho) + eps;",
            "B[i * mk + j] = Pi1[i * mk + j] * (exp(Lam[i * mk + j] / rho) + eps);", 1,
            "X3: eps inside the product in Eq.badmmc1b"),
    "M15": (ORC, "C[b + i * mk + j] = D[(size_t)xs[i] * V + ys[off[k] + j]];",
            "C[b + i * mk + j] = D[(size_t)ys[off[k] + j] * V + xs[i]];", 1, "symbolic table transposed"),
    "M16": (ORC, "double rho = rho0 * sumC / ((double)m * (double)n);",
            "double rho = rho0 * sumC / ((double)m * (double)n * (double)N);", 2, "X1 in the symbolic mode"),
    "M17": (ORC, "exp(Lam[i * mk + j] / rho) + eps;", "exp(-Lam[i * mk + j] / rho) + eps;", 1,
            "Eq.badmmc1b exp sign"),
    "M18": (ORC, "c += diff * diff;", "c += fabs(diff);", 1, "ground cost not squared"),
    "M19": (ORC, "Pi2[b + i * mk + j] = w[i] * omega[off[k] + j];", "Pi2[b + i * mk + j] = omega[off[k] + j] / m;", 1,
            "product init ignores w0"),
    "M20": (ORC, "if (Pi2_warm && warm_mask && warm_mask[k])\n", "if (0)\n", 1, "warm start ignored"),
    "M21": (ORC, "if (x && t % tau == 0 && status == AD2O_OK)", "if (x && (t - 1) % tau == 0 && status == AD2O_OK)", 1,
            "X6: support update at the wrong iteration"),
    "M22": (ORC, "for (int t = 0; t < d; ++t) num[t] += p * Y[(off[k] + j) * d + t];",
            "for (int t = 0; t < d; ++t) num[t] += p * Y[(off[k] + (j + 1) % mk) * d + t];", 1,
            "Eq.updatex member point index"),
    "M23": (ORC, "s /= (double)N;\n        w[i] = (rule == 1) ? s * s : s;",
            "s /= (double)N;\n        w[i] = (rule == 1) ? s : s * s;", 1, "R1/R2 swapped"),
    "M24": (OT, "if (W < b1) {", "if (W <= b1) {", 1, "X13: ties to the highest index"),
    "M25": (OT, "s += df * df;", "s += fabs(df);", 1, "W^2 cost not squared"),
    "M26": (OT, "x[bi * d + t] = (w[bi] * x[bi * d + t] + w[bj] * x[bj * d + t]) / wb;",
            "x[bi * d + t] = (x[bi * d + t] + x[bj * d + t]) / 2;", 1, "Eq.merge unweighted mean"),
    # initial partition (oracle/seed.py, X20-X23)
    "S1": (SEED, 'side="right"', 'side="left"', 1, "X20: D^2 draw on the prefix boundary (left)"),
    "S2": (SEED, "d2 = np.minimum(d2, sq_dist(P, centres[c]))", "d2 = sq_dist(P, centres[c])", 1,
           "D^2 to the newest centre only"),
    "S3": (SEED, "acc = acc + diff * diff", "acc = acc + np.abs(diff)", 1, "distance not squared"),
    "S4": (SEED, "return np.argmin(D, axis=1).astype(np.int32)",
           "return (D.shape[1] - 1 - np.argmin(D[:, ::-1], axis=1)).astype(np.int32)", 1, "ties to the highest index"),
    "S5": (SEED, "centres[cnt > 0, t] = s[cnt > 0] / cnt[cnt > 0]", "centres[cnt > 0, t] = s[cnt > 0] / cnt.sum()", 1,
           "Lloyd centre divided by the wrong count"),
    "S6": (SEED, "dist[counts[lab] <= 1] = -1.0", "", 1, "repair may empty a singleton cluster"),
    "S7": (SEED, "k = int(np.argmax(dist))", "k = int(np.argmin(np.where(dist < 0, np.inf, dist)))", 1,
           "repair takes the nearest member"),
    "S8": (SEED, "mu[has] = mu[has] + om[idx, None] * Y[idx]", "mu[has] = mu[has] + Y[idx] / mk[has, None]", 1,
           "unweighted member means"),
    "S9": (SEED, "pick[c] = big[min(int(u[c] * len(big)), len(big) - 1)]", "pick[c] = big[0]", 1,
           "X23: the draw ignored"),
    "S10": (SEED, "centres[0] = P[min(int(u[0] * ns), ns - 1)]", "centres[0] = P[0]", 1, "X20: first draw ignored"),
}


# tests that compare the oracle with itself (another mode or thread count): they catch some of the
# mutations but pin nothing against the paper, so a mutation must be killed without them
SELF_REFERENTIAL = ["test_symbolic_table_equals_euclidean_with_fixed_support",
                    "test_oracle_thread_count_does_not_change_results"]


def mutate(src: str, old: str, new: str, occ: int) -> str:
    pos = -1
    for _ in range(occ):
        pos = src.find(old, pos + 1)
        if pos < 0:
            raise KeyError(old)
    return src[:pos] + new + src[pos + len(old):]


def run(ids):
    rows = []
    for mid in ids:
        f, old, new, occ, what = MUTATIONS[mid]
        with tempfile.TemporaryDirectory(prefix=f"mut{mid}_") as tmp:
            for d in ("oracle", "tests", "paper_1510_00012_b200"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__", "csrc"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            p = os.path.join(tmp, f)
            src = open(p).read()
            open(p, "w").write(mutate(src, old, new, occ))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "tests/test_oracle_pins.py", "tests/test_oracle_seed_pins.py"] + [f"--deselect=tests/test_oracle_pins.py::{t}" for t in SELF_REFERENTIAL],
                               cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            first = ""
            for ln in r.stdout.splitlines():
                if ln.startswith("FAILED"):
                    first = ln.split("::", 1)[1].split(" ")[0]
                    break
            rows.append((mid, what, "killed" if killed else "SURVIVED", first))
            print(f"{mid:4s} {what:55s} {'killed' if killed else 'SURVIVED':9s} {first}", flush=True)
    return rows


if __name__ == "__main__":
    ids = sys.argv[1:] or list(MUTATIONS)
    rows = run(ids)
    sys.exit(1 if any(r[2] == "SURVIVED" for r in rows) else 0)
