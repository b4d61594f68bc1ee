"""fp64 CPU ORACLE for the modified B-ADMM barycenter path (arXiv 1510.00012, Alg. 4).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_1510_00012_b200`` never imports it and shares no code with it (the only common
module is the seeded input generator ``paper_1510_00012_b200.workloads``, which holds none
of the method's arithmetic).

The arithmetic lives in plain C (``ad2_oracle.c``: Alg. 4 and its closed forms,
``ad2_oracle_ot.c``: exact transport by the transportation simplex); this module compiles it
with gcc (``-O2 -fopenmp``, no fast-math) and exposes thin ctypes wrappers.  Matrices are
row-major m x m_k per member (the paper's Pi^(k) in R^{m x m_k}).

Parity status of each function is recorded in DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "ad2_oracle.c"), os.path.join(_HERE, "ad2_oracle_ot.c")]
_SO = os.path.join(_HERE, "libad2_oracle.so")
_lock = threading.Lock()
_lib = None

ERR = {0: "ok", 1: "arg", 2: "zero_rho", 3: "nonfinite", 4: "oom"}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, fp64, no fast-math)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp] + _SRCS + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            d, i, p, i64 = C.c_double, C.c_int, C.c_void_p, C.c_int64
            L.ad2o_assign.argtypes = [i, i, i, p, p, i, p, p, p, p, p, p]
            L.ad2o_badmm_table.argtypes = [i, i, p, p, p, p, p, p, i, p, p, i, i, d, d, d, p, p, p, p, p]
            L.ad2o_merge.argtypes = [i, i, p, p, i, p, p]
            L.ad2o_cost.argtypes = [i, i, i, p, p, p]
            L.ad2o_rho.argtypes = [i, i, p, i, p, p, d, p]
            L.ad2o_rho.restype = d
            L.ad2o_pi1.argtypes = [i, i, p, p, p, p, d, d, p]
            L.ad2o_pi1_tilde.argtypes = [i, i, p, p, d, d, p]
            L.ad2o_rowmass.argtypes = [i, i, p, p, p]
            L.ad2o_consensus.argtypes = [i, i, p, i, p]
            L.ad2o_pi2.argtypes = [i, i, p, p, p]
            L.ad2o_dual.argtypes = [i, i, p, p, p, d]
            L.ad2o_update_support.argtypes = [i, i, p, p, i, p, p, p]
            L.ad2o_surrogate.argtypes = [i, i, p, i, p, p, p]
            L.ad2o_surrogate.restype = d
            L.ad2o_badmm_centroid.argtypes = [i, i, i, p, p, p, p, p, p, p, i, i, i, d, d, d,
                                              p, p, p, p, p, i]
            L.ad2o_badmm_centroid.restype = i
            L.ad2o_transport.argtypes = [i, i, p, p, p, p, p]
            L.ad2o_transport.restype = d
            L.ad2o_w2sq.argtypes = [i, i, i, p, p, p, p, p]
            L.ad2o_w2sq.restype = d
            L.ad2o_exact_objective.argtypes = [i, i, p, p, i, p, p, p]
            L.ad2o_exact_objective.restype = d
            L.ad2o_max_threads.restype = i
            _lib = L
        return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def max_threads() -> int:
    return int(lib().ad2o_max_threads())


# ---- single-formula wrappers (each cites its equation in ad2_oracle.c) ----

def cost(x, y) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    m, d = x.shape
    mk = y.shape[0]
    out = np.empty((m, mk))
    lib().ad2o_cost(m, mk, d, _ptr(x), _ptr(y), _ptr(out))
    return out


def rho(x, offsets, Y, rho0=2.0) -> float:
    x, Y = _f64(x), _f64(Y)
    off = np.ascontiguousarray(offsets, np.int64)
    return float(lib().ad2o_rho(x.shape[0], x.shape[1], _ptr(x), len(off) - 1, _ptr(off), _ptr(Y), rho0, None))


def pi1(Pi2, Lam, Cm, omega, rho_, eps=1e-16) -> np.ndarray:
    Pi2, Lam, Cm, omega = map(_f64, (Pi2, Lam, Cm, omega))
    m, mk = Pi2.shape
    out = np.empty((m, mk))
    lib().ad2o_pi1(m, mk, _ptr(Pi2), _ptr(Lam), _ptr(Cm), _ptr(omega), rho_, eps, _ptr(out))
    return out


def pi1_tilde(Pi1, Lam, rho_, eps=1e-16) -> np.ndarray:
    Pi1, Lam = _f64(Pi1), _f64(Lam)
    m, mk = Pi1.shape
    out = np.empty((m, mk))
    lib().ad2o_pi1_tilde(m, mk, _ptr(Pi1), _ptr(Lam), rho_, eps, _ptr(out))
    return out


def rowmass(B):
    B = _f64(B)
    m, mk = B.shape
    r, wt = np.empty(m), np.empty(m)
    lib().ad2o_rowmass(m, mk, _ptr(B), _ptr(r), _ptr(wt))
    return r, wt


def consensus(wt, rule=0) -> np.ndarray:
    wt = _f64(wt)
    N, m = wt.shape
    out = np.empty(m)
    lib().ad2o_consensus(N, m, _ptr(wt), int(rule), _ptr(out))
    return out


def pi2(B, w) -> np.ndarray:
    B, w = _f64(B), _f64(w)
    m, mk = B.shape
    out = np.empty((m, mk))
    lib().ad2o_pi2(m, mk, _ptr(B), _ptr(w), _ptr(out))
    return out


def dual(Lam, Pi1, Pi2, rho_) -> np.ndarray:
    Lam = _f64(Lam).copy()
    Pi1, Pi2 = _f64(Pi1), _f64(Pi2)
    m, mk = Lam.shape
    lib().ad2o_dual(m, mk, _ptr(Lam), _ptr(Pi1), _ptr(Pi2), rho_)
    return Lam


def update_support(x, w, offsets, Y, Pi2_list) -> np.ndarray:
    x = _f64(x).copy()
    w, Y = _f64(w), _f64(Y)
    off = np.ascontiguousarray(offsets, np.int64)
    cat = np.concatenate([_f64(P).ravel() for P in Pi2_list])
    m, d = x.shape
    lib().ad2o_update_support(m, d, _ptr(x), _ptr(w), len(off) - 1, _ptr(off), _ptr(Y), _ptr(cat))
    return x


def transport(a, b, c, want_plan=False):
    a, b, c = _f64(a), _f64(b), _f64(c)
    ma, mb = c.shape
    plan = np.empty((ma, mb)) if want_plan else None
    it = C.c_int(0)
    W = lib().ad2o_transport(ma, mb, _ptr(a), _ptr(b), _ptr(c), _ptr(plan) if plan is not None else None,
                             C.byref(it))
    return (W, plan) if want_plan else W


def w2sq(xa, wa, xb, wb) -> float:
    xa, wa, xb, wb = map(_f64, (xa, wa, xb, wb))
    return float(lib().ad2o_w2sq(len(wa), len(wb), xa.shape[1], _ptr(xa), _ptr(wa), _ptr(xb), _ptr(wb), None))


def exact_objective(x, w, offsets, Y, omega) -> float:
    """Eq.centroid by exact OT, member weights renormalised as in O1."""
    x, w, Y, omega = map(_f64, (x, w, Y, omega))
    off = np.ascontiguousarray(offsets, np.int64)
    om = omega / np.repeat(np.add.reduceat(omega, off[:-1] - off[0]), np.diff(off))
    w = w / w.sum()
    return float(lib().ad2o_exact_objective(x.shape[0], x.shape[1], _ptr(x), _ptr(w), len(off) - 1,
                                            _ptr(off - off[0]), _ptr(Y), _ptr(om)))


def assign(x, w, offsets, Y, omega):
    """Assignment step (Alg. 1; O7, X13): exact W^2 of every member to every centroid
    (transportation simplex, no pruning), label = argmin with ties to the lowest index.
    Returns (labels int32 [N], best W^2 [N], second-best W^2 [N])."""
    x, w, Y, omega = map(_f64, (x, w, Y, omega))
    K, m, d = x.shape
    off = np.ascontiguousarray(offsets, np.int64)
    off = off - off[0]
    N = len(off) - 1
    lab = np.zeros(N, np.int32)
    best = np.zeros(N)
    second = np.zeros(N)
    lib().ad2o_assign(K, m, d, _ptr(x), _ptr(w), N, _ptr(off), _ptr(Y), _ptr(omega), lab.ctypes.data,
                      _ptr(best), _ptr(second))
    return lab, best, second


# ---- Algorithm 4 ----

class Result:
    __slots__ = ("x", "w", "Pi1", "Pi2", "Lam", "rho", "obj", "mats")

    def member(self, name: str, k: int) -> np.ndarray:
        """Row-major m x m_k matrix of member k from the concatenated output."""
        return self.mats[name][k]


def badmm_centroid(x0, w0, offsets, Y, omega, T, tau, rule=0, rho0=2.0, eps=1e-16, wtol=1e-6,
                   warm=None, warm_mask=None, nthreads=0, want_state=True) -> Result:
    """Alg. 4 for one cluster; see ad2o_badmm_centroid in ad2_oracle.c."""
    x = _f64(x0).copy()
    w = _f64(w0).copy()
    Y, omega = _f64(Y), _f64(omega)
    off = np.ascontiguousarray(offsets, np.int64)
    m, d = x.shape
    N = len(off) - 1
    E = m * int(off[-1] - off[0])
    Pi1 = np.empty(E) if want_state else None
    Pi2 = np.empty(E) if want_state else None
    Lam = np.empty(E) if want_state else None
    r = C.c_double(0.0)
    obj = C.c_double(0.0)
    warm_cat = None
    wm = None
    if warm is not None:
        warm_cat = np.concatenate([_f64(P).ravel() for P in warm])
        wm = np.ascontiguousarray(warm_mask if warm_mask is not None else np.ones(N), np.uint8)
    st = lib().ad2o_badmm_centroid(
        m, d, N, _ptr(off), _ptr(Y), _ptr(omega), _ptr(x), _ptr(w),
        _ptr(warm_cat) if warm_cat is not None else None, _ptr(wm) if wm is not None else None,
        int(T), int(tau), int(rule), float(rho0), float(eps), float(wtol),
        _ptr(Pi1) if want_state else None, _ptr(Pi2) if want_state else None,
        _ptr(Lam) if want_state else None, C.byref(r), C.byref(obj), int(nthreads))
    if st != 0:
        raise OracleError(f"ad2o_badmm_centroid: {ERR.get(st, st)}")
    res = Result()
    res.x, res.w, res.rho, res.obj = x, w, r.value, obj.value
    res.Pi1, res.Pi2, res.Lam = Pi1, Pi2, Lam
    res.mats = {}
    if want_state:
        sizes = np.diff(off)
        bounds = np.concatenate([[0], np.cumsum(m * sizes)])
        for name, cat in (("Pi1", Pi1), ("Pi2", Pi2), ("Lam", Lam)):
            res.mats[name] = [cat[bounds[k]:bounds[k + 1]].reshape(m, sizes[k]) for k in range(N)]
    return res


def run_bundle(bundle, T=None, tau=None, rule=None, clusters=None, nthreads=0, want_state=True,
               warm=None):
    """Run Alg. 4 independently on every cluster of a workloads.Bundle (clusters are
    independent within a round).  Returns {c: Result} and the member lists."""
    s = bundle.sched
    T = s.T if T is None else T
    tau = s.tau if tau is None else tau
    rule = s.rule if rule is None else rule
    wtol = 1e-6 if bundle.dtype == "f64" else 1e-5
    out, members = {}, {}
    for c in (range(bundle.K) if clusters is None else clusters):
        mem = np.nonzero(bundle.labels == c)[0]
        members[c] = mem
        sub = bundle.subset(mem)
        out[c] = badmm_centroid(bundle.x0[c], bundle.w0[c], sub.offsets, sub.supports, sub.weights,
                                T, tau, rule, s.rho0, s.eps, wtol, nthreads=nthreads,
                                want_state=want_state)
    return out, members


def cluster(bundle, T, tau, max_rounds, stop_frac=0.0, rule=None):
    """The AD2 outer loop (Alg. 1) with Alg. 4 as the centroid update, as SURVEY.md
    §8(c) O8 fixes it: each round = Alg. 4 per cluster from the current centroids (warm Pi^(2)
    for members whose label did not change; Lambda reset, X7) -> exact assignment
    (``assign``, lowest index on ties); stop after max_rounds or when the changed fraction
    <= stop_frac.  Returns (labels, rounds, changed fractions, per-round surrogate objectives
    [rounds][K], final x, final w)."""
    s = bundle.sched
    rule = s.rule if rule is None else rule
    wtol = 1e-6 if bundle.dtype == "f64" else 1e-5
    K = bundle.K
    lab = np.asarray(bundle.labels, np.int32).copy()
    x, w = _f64(bundle.x0).copy(), _f64(bundle.w0).copy()
    prev_pi2, warm_ok = {}, np.zeros(bundle.N, bool)
    changed, objs = [], []
    rounds = 0
    for r in range(max_rounds):
        nx, nw, pi2 = x.copy(), w.copy(), {}
        obj = np.zeros(K)
        for c in range(K):
            mem = np.nonzero(lab == c)[0]
            if len(mem) == 0:
                raise OracleError(f"cluster {c} empty in round {r}")
            sub = bundle.subset(mem)
            wm = warm_ok[mem] if r > 0 else None
            warm = [prev_pi2[k] if warm_ok[k] else np.zeros((bundle.m, int(bundle.offsets[k + 1] - bundle.offsets[k])))
                    for k in mem] if r > 0 else None
            res = badmm_centroid(x[c], w[c], sub.offsets, sub.supports, sub.weights, T, tau, rule, s.rho0, s.eps,
                                 wtol, warm=warm, warm_mask=wm)
            nx[c], nw[c], obj[c] = res.x, res.w, res.obj
            for k, P in zip(mem, res.mats["Pi2"]):
                pi2[k] = P
        x, w = nx, nw
        objs.append(obj)
        new, _, _ = assign(x, w, bundle.offsets, bundle.supports, bundle.weights)
        warm_ok = new == lab
        changed.append(float(np.mean(new != lab)))
        lab, prev_pi2 = new, pi2
        rounds = r + 1
        if changed[-1] <= stop_frac:
            break
    return lab, rounds, np.array(changed), np.array(objs), x, w


def badmm_table(xs, w0, offsets, ys, omega, D, T, rule=0, rho0=2.0, eps=1e-16, wtol=1e-6, warm=None,
                warm_mask=None, want_state=True) -> Result:
    """Alg. 4 on symbolic supports: C^(k)_ij = D[xs_i, ys_j] from the cost table, the
    support update skipped (fixed symbols).  xs int [m], ys int [n], D [V][V]."""
    xs = np.ascontiguousarray(xs, np.int32)
    ys = np.ascontiguousarray(ys, np.int32)
    w = _f64(w0).copy()
    omega, D = _f64(omega), _f64(D)
    off = np.ascontiguousarray(offsets, np.int64)
    m, N, V = len(xs), len(off) - 1, D.shape[0]
    E = m * int(off[-1] - off[0])
    Pi1, Pi2, Lam = (np.empty(E), np.empty(E), np.empty(E)) if want_state else (None, None, None)
    r, obj = C.c_double(0.0), C.c_double(0.0)
    warm_cat = wm = None
    if warm is not None:
        warm_cat = np.concatenate([_f64(P).ravel() for P in warm])
        wm = np.ascontiguousarray(warm_mask if warm_mask is not None else np.ones(N), np.uint8)
    st = lib().ad2o_badmm_table(m, N, _ptr(off), _ptr(ys), _ptr(omega), _ptr(xs), _ptr(w), _ptr(D), V,
                                _ptr(warm_cat) if warm_cat is not None else None, _ptr(wm) if wm is not None else None,
                                int(T), int(rule), float(rho0), float(eps), float(wtol),
                                _ptr(Pi1) if want_state else None, _ptr(Pi2) if want_state else None,
                                _ptr(Lam) if want_state else None, C.byref(r), C.byref(obj))
    if st != 0:
        raise OracleError(f"ad2o_badmm_table: {ERR.get(st, st)}")
    res = Result()
    res.x, res.w, res.rho, res.obj = xs.copy(), w, r.value, obj.value
    res.mats = {}
    if want_state:
        sizes = np.diff(off)
        bounds = np.concatenate([[0], np.cumsum(m * sizes)])
        for name, cat in (("Pi1", Pi1), ("Pi2", Pi2), ("Lam", Lam)):
            res.mats[name] = [cat[bounds[k]:bounds[k + 1]].reshape(m, sizes[k]) for k in range(N)]
    return res


def merge(y, w, m):
    """Eq.merge initialisation of a centroid with m points from one member."""
    y, w = _f64(y), _f64(w)
    mk, d = y.shape
    x = np.empty((m, d))
    wo = np.empty(m)
    lib().ad2o_merge(mk, d, _ptr(y), _ptr(w), m, _ptr(x), _ptr(wo))
    return x, wo
