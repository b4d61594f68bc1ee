"""Thin ctypes binding of libad2 (include/ad2.h) — argument marshalling only.

Every arithmetic step runs in the CUDA kernels of ``libad2.so``.  There is no CPU fallback: if
the library is missing or no CUDA device is present, the calls raise ``RuntimeError``.

Arrays may be torch tensors (CUDA tensors for ``mem="device"``, CPU — ideally pinned — tensors
for ``mem="host"``) or numpy arrays (host).  Names follow the paper:
``offsets``/``supports``/``weights`` = the ragged members P^(k), ``labels`` = l^(k),
``x``/``w`` = centroid support points and weights, Pi1/Pi2/Lambda = the B-ADMM state.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# AD2_LIB selects another build of the same library (e.g. libad2_checked.so, device assertions on)
LIB_PATH = os.environ.get("AD2_LIB") or os.path.join(_HERE, "libad2.so")

F32, F64 = 0, 1
R1, R2 = 0, 1
DEVICE, HOST = 0, 1
PI1, PI2, LAMBDA, COST = 0, 1, 2, 3
COST_FP32, COST_TC_BF16, COST_TABLE = 0, 1, 2

STATUS = {0: "ok", 1: "ARG", 2: "OOM", 3: "CUDA", 4: "NCCL", 5: "NONFINITE", 6: "ZERO_RHO", 7: "EMPTY",
          8: "STATE"}


class AD2Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"AD2_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


class Batch(C.Structure):
    _fields_ = [("dtype", C.c_int), ("mem", C.c_int), ("d", C.c_int32), ("m", C.c_int32), ("K", C.c_int32),
                ("n_members", C.c_int64), ("offsets", C.c_void_p), ("supports", C.c_void_p),
                ("weights", C.c_void_p), ("labels", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("rho0", C.c_double), ("eps", C.c_double), ("rule", C.c_int32), ("cost_mode", C.c_int32)]


class Loop(C.Structure):
    _fields_ = [("T", C.c_int32), ("tau", C.c_int32), ("max_rounds", C.c_int32), ("stop_frac", C.c_double)]


class Info(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("dtype", C.c_int32), ("d", C.c_int32), ("m", C.c_int32),
                ("K", C.c_int32), ("n_members", C.c_int64), ("n_points", C.c_int64), ("entries", C.c_int64),
                ("n_items", C.c_int64), ("variant", C.c_int32), ("mp", C.c_int32), ("nch", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("launches", C.c_int64),
                ("state_bytes", C.c_int64), ("state_mode", C.c_int32), ("eps_floor_columns", C.c_int32),
                ("assign_certified", C.c_int64), ("assign_exact", C.c_int64), ("tc_cost", C.c_int32)]


EXPORTS = ["ad2_create", "ad2_nccl_unique_id", "ad2_attach_nccl", "ad2_barycenter_init", "ad2_badmm_step",
           "ad2_update_support", "ad2_objective", "ad2_get_centroids", "ad2_get_plans", "ad2_get_rho",
           "ad2_get_info", "ad2_set_profiling", "ad2_prof_read", "ad2_assign", "ad2_assign_symbolic",
           "ad2_set_cost_table", "ad2_cluster", "ad2_merge_init", "ad2_kmeanspp", "ad2_label_nearest",
           "ad2_pick_members", "ad2_prefetch", "ad2_sync",
           "ad2_set_state_mode", "ad2_set_tc_cost", "ad2_group_open", "ad2_group_allreduce", "ad2_attach_group", "ad2_group_close",
           "ad2_last_error",
           "ad2_status_string", "ad2_destroy"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libad2.so (RuntimeError if it has not been built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libad2.so not built at {path}; run `python -m paper_1510_00012_b200.build`")
    L = C.CDLL(path)
    p, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    L.ad2_create.argtypes = [C.POINTER(p), C.c_int, p]
    L.ad2_nccl_unique_id.argtypes = [p]
    L.ad2_attach_nccl.argtypes = [p, C.c_int, C.c_int, p]
    L.ad2_barycenter_init.argtypes = [p, C.POINTER(Batch), C.POINTER(Params), p, p, p, p]
    L.ad2_badmm_step.argtypes = [p, i32]
    L.ad2_update_support.argtypes = [p]
    L.ad2_objective.argtypes = [p, p]
    L.ad2_get_centroids.argtypes = [p, p, p, C.c_int]
    L.ad2_get_plans.argtypes = [p, C.c_int, p, C.c_int]
    L.ad2_get_rho.argtypes = [p, p]
    L.ad2_get_info.argtypes = [p, C.POINTER(Info)]
    L.ad2_set_profiling.argtypes = [p, C.c_int]
    L.ad2_prof_read.argtypes = [p, p, i64, C.POINTER(i64), C.POINTER(d)]
    L.ad2_assign.argtypes = [p, C.POINTER(Batch), p, p, p, p, C.c_int, C.POINTER(i64)]
    L.ad2_assign_symbolic.argtypes = [p, C.POINTER(Batch), p, p, p, p, C.c_int, C.POINTER(i64)]
    L.ad2_set_cost_table.argtypes = [p, p, i32, C.c_int, C.c_int]
    L.ad2_cluster.argtypes = [p, C.POINTER(Batch), C.POINTER(Params), C.POINTER(Loop), p, p, p, C.POINTER(i32),
                              p, p]
    L.ad2_merge_init.argtypes = [p, C.POINTER(Batch), p, p, p, C.c_int]
    L.ad2_kmeanspp.argtypes = [p, C.POINTER(Batch), p, i64, p, i32, p, C.c_int]
    L.ad2_label_nearest.argtypes = [p, C.POINTER(Batch), p, p, p, C.c_int]
    L.ad2_pick_members.argtypes = [p, C.POINTER(Batch), p, p]
    L.ad2_prefetch.argtypes = [p, C.POINTER(Batch), C.c_int]
    L.ad2_sync.argtypes = [p]
    L.ad2_last_error.argtypes = [p]
    L.ad2_last_error.restype = C.c_char_p
    L.ad2_status_string.argtypes = [C.c_int]
    L.ad2_status_string.restype = C.c_char_p
    L.ad2_destroy.argtypes = [p]
    L.ad2_destroy.restype = None
    L.ad2_set_state_mode.argtypes = [p, i32]
    L.ad2_set_tc_cost.argtypes = [p, i32]
    L.ad2_group_open.argtypes = [C.POINTER(p), C.c_char_p, C.c_int, C.c_int, i64]
    L.ad2_group_allreduce.argtypes = [p, p, i64, i32]
    L.ad2_attach_group.argtypes = [p, p]
    L.ad2_group_close.argtypes = [p]
    L.ad2_group_close.restype = None
    for f in EXPORTS:
        if f not in ("ad2_last_error", "ad2_status_string", "ad2_destroy", "ad2_group_close"):
            getattr(L, f).restype = C.c_int
    _lib = L
    return L


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(type(a))


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = C.create_string_buffer(128)
    st = L.ad2_nccl_unique_id(buf)
    if st != 0:
        raise AD2Error(st, "ncclGetUniqueId failed / NCCL not loadable")
    return buf.raw


GROUP_F32, GROUP_F64, GROUP_U64 = 0, 1, 2


class Group:
    """Host process group (ad2_group_open): ranks that are processes on one host sum libad2's
    per-cluster partials through POSIX shared memory instead of NCCL.  Collective: every rank
    opens the same `name` ("/...") with the same nranks."""

    def __init__(self, name: str, nranks: int, rank: int, slot_bytes: int = 64 << 20):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.ad2_group_open(C.byref(h), name.encode(), int(nranks), int(rank), int(slot_bytes))
        if st != 0:
            raise AD2Error(st, f"ad2_group_open({name!r}, {nranks}, {rank}) failed")
        self.h = h
        self.nranks, self.rank = nranks, rank

    def allreduce(self, a: np.ndarray) -> np.ndarray:
        """In-place sum of a host array over the group (rank order)."""
        dt = {np.dtype(np.float32): GROUP_F32, np.dtype(np.float64): GROUP_F64,
              np.dtype(np.uint64): GROUP_U64}[a.dtype]
        st = self.L.ad2_group_allreduce(self.h, _ptr(a), a.size, dt)
        if st != 0:
            raise AD2Error(st, "ad2_group_allreduce failed")
        return a

    def close(self):
        if getattr(self, "h", None):
            self.L.ad2_group_close(self.h)
            self.h = None


class Context:
    """One B-ADMM barycenter context on one GPU (one per rank)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.ad2_create(C.byref(h), int(device), C.c_void_p(stream) if stream else None)
        if st != 0:
            raise AD2Error(st, "ad2_create failed (no CUDA device?)")
        self.h = h
        self.K = self.m = self.d = None
        self.dtype = None
        self._keep = []

    def _chk(self, st: int):
        if st != 0:
            raise AD2Error(st, self.L.ad2_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.ad2_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def attach_nccl(self, nranks: int, rank: int, unique_id: bytes):
        self._chk(self.L.ad2_attach_nccl(self.h, nranks, rank, C.c_char_p(unique_id)))

    def attach_group(self, group: "Group"):
        self._chk(self.L.ad2_attach_group(self.h, group.h))
        self._keep.append(group)                # the group must outlive the context

    def init(self, offsets, supports, weights, labels, x0, w0, K: int, m: int, rho0=2.0, eps=1e-16,
             rule=R1, warm_mask=None, mem: str = "device", dtype: Optional[str] = None,
             cost_mode: int = 0) -> np.ndarray:
        """ad2_barycenter_init; returns rho per cluster (host float64 [K])."""
        if dtype is None:
            dt = getattr(weights, "dtype", None)
            dtype = "f64" if str(dt) in ("float64", "torch.float64") else "f32"
        if cost_mode == COST_TABLE or len(supports.shape) == 1:
            d = 1                                             # symbolic supports: int32 ids
        else:
            d = int(supports.shape[1]) if supports.shape[0] > 0 else int(x0.shape[-1])
        self.table = cost_mode == COST_TABLE
        b = Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, d, int(m), int(K),
                  int(len(labels)), _ptr(offsets), _ptr(supports), _ptr(weights), _ptr(labels))
        prm = Params(float(rho0), float(eps), int(rule), int(cost_mode))
        wm = None
        if warm_mask is not None:
            wm = np.ascontiguousarray(np.asarray(warm_mask), dtype=np.uint8)
        rho = np.zeros(int(K))
        self._chk(self.L.ad2_barycenter_init(self.h, C.byref(b), C.byref(prm), _ptr(x0), _ptr(w0),
                                             _ptr(wm), rho.ctypes.data))
        self.K, self.m, self.d, self.dtype = int(K), int(m), d, dtype
        self._offsets = offsets
        self._offsets_host = None
        return rho

    def prefetch(self, offsets, supports, weights, labels, dtype: Optional[str] = None, cost_mode: int = 0):
        """ad2_prefetch: start the host->device copies of a host batch on the context's copy stream;
        the next init(..., mem="host") with the same arrays uses them (pinned arrays overlap)."""
        if dtype is None:
            dt = getattr(weights, "dtype", None)
            dtype = "f64" if str(dt) in ("float64", "torch.float64") else "f32"
        d = 1 if (cost_mode == COST_TABLE or len(supports.shape) == 1) else int(supports.shape[1])
        b = Batch(F64 if dtype == "f64" else F32, HOST, d, 1, 1, int(len(labels)), _ptr(offsets), _ptr(supports),
                  _ptr(weights), _ptr(labels))
        self._chk(self.L.ad2_prefetch(self.h, C.byref(b), int(cost_mode)))

    @property
    def offsets_host(self) -> np.ndarray:
        if self._offsets_host is None:
            o = self._offsets
            self._offsets_host = np.asarray(o.cpu() if hasattr(o, "cpu") else o)
        return self._offsets_host

    def step(self, n_iters: int):
        self._chk(self.L.ad2_badmm_step(self.h, int(n_iters)))

    def update_support(self):
        self._chk(self.L.ad2_update_support(self.h))

    def objective(self) -> np.ndarray:
        out = np.zeros(self.K)
        self._chk(self.L.ad2_objective(self.h, out.ctypes.data))
        return out

    def _np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    def centroids(self):
        """(x [K][m][d], w [K][m]); symbolic rounds return the centroid symbol ids x [K][m] (int32)."""
        if getattr(self, "table", False):
            x = np.empty((self.K, self.m), np.int32)
        else:
            x = np.empty((self.K, self.m, self.d), self._np_dtype())
        w = np.empty((self.K, self.m), self._np_dtype())
        self._chk(self.L.ad2_get_centroids(self.h, x.ctypes.data, w.ctypes.data, HOST))
        return x, w

    def centroids_into(self, x, w, mem: str = "device"):
        self._chk(self.L.ad2_get_centroids(self.h, _ptr(x), _ptr(w), HOST if mem == "host" else DEVICE))

    def plans(self, which: int) -> np.ndarray:
        """Concatenated member blocks in caller order, column-major m x m_k each."""
        n = int(self.offsets_host[-1])
        out = np.empty(self.m * n, self._np_dtype())
        self._chk(self.L.ad2_get_plans(self.h, int(which), out.ctypes.data, HOST))
        return out

    def member_matrices(self, which: int):
        """List of m x m_k matrices (row i = centroid point, col j = member point)."""
        cat = self.plans(which)
        off = self.offsets_host
        m = self.m
        return [cat[m * off[k]: m * off[k + 1]].reshape(off[k + 1] - off[k], m).T for k in range(len(off) - 1)]

    def rho(self) -> np.ndarray:
        out = np.zeros(self.K)
        self._chk(self.L.ad2_get_rho(self.h, out.ctypes.data))
        return out

    def info(self) -> dict:
        i = Info()
        self._chk(self.L.ad2_get_info(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in Info._fields_}

    def set_tc_cost(self, enable: int):
        """ad2_set_tc_cost: 1 tensor-core dot products in the variant-2 cost (default), 0 FFMA2."""
        self._chk(self.L.ad2_set_tc_cost(self.h, int(enable)))

    def set_state_mode(self, mode: int):
        """ad2_set_state_mode: 0 exact Pi1/Lambda streaming, 1 epoch-anchored compressed state."""
        self._chk(self.L.ad2_set_state_mode(self.h, int(mode)))

    def set_profiling(self, enable):
        """ad2_set_profiling: False/0 off, True/1 every later step, 2 the next step only."""
        self._chk(self.L.ad2_set_profiling(self.h, int(enable)))

    def prof_read(self):
        """(per-launch ms of the last profiled step's iteration kernels, step ms)."""
        buf = np.zeros(4096)
        n, step = C.c_int64(), C.c_double()
        self._chk(self.L.ad2_prof_read(self.h, buf.ctypes.data, len(buf), C.byref(n), C.byref(step)))
        return buf[:min(n.value, len(buf))].copy(), step.value

    def assign(self, offsets, supports, weights, x, w, mem: str = "device", dtype: Optional[str] = None):
        """ad2_assign: exact-W2 labels of the members against centroids (x [K][m][d], w [K][m]).
        Returns (labels int32 [N], W2 float64 [N], number of exact transport solves) on the host."""
        if dtype is None:
            dt = getattr(supports, "dtype", None)
            dtype = "f64" if str(dt) in ("float64", "torch.float64") else "f32"
        K, m, d = int(x.shape[0]), int(x.shape[1]), int(x.shape[2])
        N = int(offsets.shape[0]) - 1
        b = Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, d, m, K, N, _ptr(offsets),
                  _ptr(supports), _ptr(weights), None)
        lab = np.zeros(max(N, 0), np.int32)
        w2 = np.zeros(max(N, 0))
        n_exact = C.c_int64()
        self._chk(self.L.ad2_assign(self.h, C.byref(b), _ptr(x), _ptr(w), lab.ctypes.data, w2.ctypes.data, HOST,
                                    C.byref(n_exact)))
        return lab, w2, int(n_exact.value)

    def cluster(self, offsets, supports, weights, labels, x0, w0, K: int, m: int, T: int, tau: int,
                max_rounds: int, stop_frac: float = 0.0, rho0=2.0, eps=1e-16, rule=R1, mem: str = "device",
                dtype: Optional[str] = None, cost_mode: int = 0):
        """ad2_cluster: the AD2 outer loop on the device.  Returns a dict with the final labels
        (host int32 [N]), rounds run, changed fraction per round and surrogate objectives [rounds][K]."""
        if dtype is None:
            dt = getattr(weights, "dtype", None)
            dtype = "f64" if str(dt) in ("float64", "torch.float64") else "f32"
        d = 1 if cost_mode == COST_TABLE else int(x0.shape[-1])
        N = int(labels.shape[0])
        b = Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, d, int(m), int(K), N,
                  _ptr(offsets), _ptr(supports), _ptr(weights), _ptr(labels))
        prm = Params(float(rho0), float(eps), int(rule), int(cost_mode))
        lp = Loop(int(T), int(tau), int(max_rounds), float(stop_frac))
        changed = np.zeros(max_rounds)
        obj = np.zeros((max_rounds, int(K)))
        rounds = C.c_int32()
        if mem == "host":
            lab = np.zeros(N, np.int32)
            out = lab.ctypes.data
        else:
            import torch
            lab_t = torch.empty(N, dtype=torch.int32, device=labels.device)
            out = lab_t.data_ptr()
        self._chk(self.L.ad2_cluster(self.h, C.byref(b), C.byref(prm), C.byref(lp), _ptr(x0), _ptr(w0), out,
                                     C.byref(rounds), changed.ctypes.data, obj.ctypes.data))
        if mem != "host":
            lab = lab_t.cpu().numpy()
        self.K, self.m, self.d, self.dtype = int(K), int(m), d, dtype
        self.table = cost_mode == COST_TABLE
        self._offsets = offsets
        self._offsets_host = None
        r = rounds.value
        return {"labels": lab, "rounds": r, "changed": changed[:r], "objective": obj[:r]}

    def set_cost_table(self, D, dtype: Optional[str] = None, mem: str = "host"):
        """ad2_set_cost_table: symbol-to-symbol cost table D [V][V] for symbolic rounds."""
        if dtype is None:
            dtype = "f64" if str(getattr(D, "dtype", "")) in ("float64", "torch.float64") else "f32"
        self._chk(self.L.ad2_set_cost_table(self.h, _ptr(D), int(D.shape[0]), F64 if dtype == "f64" else F32,
                                            HOST if mem == "host" else DEVICE))

    def assign_symbolic(self, offsets, ids, weights, xs, w, mem: str = "device", dtype: Optional[str] = None):
        """ad2_assign_symbolic: labels of members (int32 symbol ids) against centroid symbols xs [K][m]."""
        if dtype is None:
            dtype = "f64" if str(getattr(weights, "dtype", "")) in ("float64", "torch.float64") else "f32"
        K, m = int(xs.shape[0]), int(xs.shape[1])
        N = int(offsets.shape[0]) - 1
        b = Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, 1, m, K, N, _ptr(offsets),
                  _ptr(ids), _ptr(weights), None)
        lab = np.zeros(max(N, 0), np.int32)
        w2 = np.zeros(max(N, 0))
        n_exact = C.c_int64()
        self._chk(self.L.ad2_assign_symbolic(self.h, C.byref(b), _ptr(xs), _ptr(w), lab.ctypes.data, w2.ctypes.data,
                                             HOST, C.byref(n_exact)))
        return lab, w2, int(n_exact.value)

    def merge_init(self, offsets, supports, weights, pick, K: int, m: int, mem: str = "device",
                   dtype: Optional[str] = None):
        """ad2_merge_init: Eq.merge centroids from the picked members; returns host (x0, w0)."""
        if dtype is None:
            dtype = "f64" if str(getattr(weights, "dtype", "")) in ("float64", "torch.float64") else "f32"
        d = int(supports.shape[1])
        N = int(offsets.shape[0]) - 1
        b = Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, d, int(m), int(K), N,
                  _ptr(offsets), _ptr(supports), _ptr(weights), None)
        pk = np.ascontiguousarray(pick, np.int64)
        ft = np.float64 if dtype == "f64" else np.float32
        x0 = np.zeros((int(K), int(m), d), ft)
        w0 = np.zeros((int(K), int(m)), ft)
        self._chk(self.L.ad2_merge_init(self.h, C.byref(b), pk.ctypes.data, x0.ctypes.data, w0.ctypes.data, HOST))
        return x0, w0

    @staticmethod
    def _seed_batch(offsets, supports, weights, labels, K, m, mem, dtype):
        if dtype is None:
            dtype = "f64" if str(getattr(weights, "dtype", "")) in ("float64", "torch.float64") else "f32"
        return Batch(F64 if dtype == "f64" else F32, HOST if mem == "host" else DEVICE, int(supports.shape[1]),
                     int(m), int(K), int(offsets.shape[0]) - 1, _ptr(offsets), _ptr(supports), _ptr(weights),
                     _ptr(labels))

    def kmeanspp(self, offsets, supports, weights, sample, u, lloyd_iters: int, mem: str = "device",
                 dtype: Optional[str] = None):
        """ad2_kmeanspp: k-means++ (X20) + Lloyd (X21) on the sampled member means; host centres [K][d]."""
        u = np.ascontiguousarray(u, np.float64)
        smp = np.ascontiguousarray(sample, np.int64)
        b = self._seed_batch(offsets, supports, weights, None, len(u), 1, mem, dtype)
        cen = np.zeros((len(u), b.d))
        self._chk(self.L.ad2_kmeanspp(self.h, C.byref(b), smp.ctypes.data, len(smp), u.ctypes.data,
                                      int(lloyd_iters), cen.ctypes.data, HOST))
        return cen

    def label_nearest(self, offsets, supports, weights, centres, mem: str = "device", dtype: Optional[str] = None):
        """ad2_label_nearest: nearest-mean labels with the empty-cluster repair (X21, X22);
        returns host (labels int32 [N], centres [K][d] after the repair)."""
        cen = np.ascontiguousarray(centres, np.float64)
        b = self._seed_batch(offsets, supports, weights, None, len(cen), 1, mem, dtype)
        lab = np.zeros(b.n_members, np.int32)
        out = np.zeros_like(cen)
        self._chk(self.L.ad2_label_nearest(self.h, C.byref(b), cen.ctypes.data, lab.ctypes.data, out.ctypes.data,
                                           HOST))
        return lab, out

    def pick_members(self, offsets, supports, weights, labels, m: int, u, mem: str = "device",
                     dtype: Optional[str] = None):
        """ad2_pick_members: the member per cluster whose support Eq.merge reduces (X23); host int64 [K]."""
        u = np.ascontiguousarray(u, np.float64)
        b = self._seed_batch(offsets, supports, weights, labels, len(u), m, mem, dtype)
        pick = np.zeros(len(u), np.int64)
        self._chk(self.L.ad2_pick_members(self.h, C.byref(b), u.ctypes.data, pick.ctypes.data))
        return pick

    def sync(self):
        self._chk(self.L.ad2_sync(self.h))


def run_schedule(ctx: Context, T: int, tau: int, before_last_step=None):
    """Alg. 4's schedule (reading X6): step(tau); update_support() per full tau block.
    before_last_step: called before the last step call (e.g. ctx.set_profiling(2))."""
    done = 0
    while done < T:
        n = min(tau, T - done)
        if before_last_step is not None and done + n >= T:
            before_last_step()
        ctx.step(n)
        done += n
        if n == tau:
            ctx.update_support()
