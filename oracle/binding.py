"""ctypes binding of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_2503_19050_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "mist_oracle.cpp")
MAX_SPLITS = 8


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, -O2 -ffp-contract=off, OpenMP)."""
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(SRC),
                                                  os.path.getmtime(os.path.join(HERE, "mist_oracle.h")))):
        return LIB_PATH
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-fPIC", "-shared", "-o", LIB_PATH + ".tmp", SRC]
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class Model(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("L", "h", "a", "k", "f", "V", "s", "e", "g", "p", "fl", "nrm")]


class ProblemS(C.Structure):
    _fields_ = [
        ("model", Model), ("B", C.c_int64), ("N", C.c_int32), ("M", C.c_int32),
        ("mem_budget", C.c_int64), ("Q", C.c_int32), ("zero_mask", C.c_int32),
        ("max_stages", C.c_int32), ("n_grad_accum", C.c_int32),
        ("grad_accum", C.POINTER(C.c_int32)),
        ("n_b", C.c_int32), ("b_values", C.POINTER(C.c_int32)),
        ("n_tp", C.c_int32), ("tp_values", C.POINTER(C.c_int32)),
        ("Tf", C.POINTER(C.c_double)), ("Tb", C.POINTER(C.c_double)),
        ("Tef", C.POINTER(C.c_double)), ("Teb", C.POINTER(C.c_double)),
        ("Thf", C.POINTER(C.c_double)), ("Thb", C.POINTER(C.c_double)),
        ("bw", (C.c_double * 2) * 4), ("lat", (C.c_double * 2) * 4),
        ("bw_h2d", C.c_double), ("bw_d2h", C.c_double),
        ("intf", (C.c_double * 4) * 16),
        ("ckpt_ends_only", C.c_int32), ("offload_off", C.c_int32),
    ]


class Group(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("G", "first", "last", "w", "l", "n", "m", "n_splits")] + [
        ("tp", C.c_int32 * MAX_SPLITS), ("dp", C.c_int32 * MAX_SPLITS), ("b", C.c_int32 * MAX_SPLITS),
        ("tuple_offset", C.c_uint64), ("config_offset", C.c_uint64), ("count", C.c_uint64)]


class Detail(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("P_layer", "P_st", "A_full", "A_bnd", "A_H", "X")] + [
        ("ch", ((C.c_double * 4) * 4) * 4), ("T", (C.c_double * 4) * 4), ("p2p", C.c_double)] + [
        (n, C.c_double) for n in ("D", "Ms", "Mwb", "Mgb", "Mob", "Ma", "Afull_D", "mem_fwd_D",
                                  "mem_bwd_D", "t", "d", "mem")] + [("feasible", C.c_int32)]


class Point(C.Structure):
    _fields_ = [("idx", C.c_uint64), ("t", C.c_double), ("y", C.c_double), ("mem", C.c_double),
                ("group", C.c_int64)]


POINT_DTYPE = np.dtype([("idx", "<u8"), ("t", "<f8"), ("y", "<f8"), ("mem", "<f8"), ("group", "<i8")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.orc_pred_intf.restype = C.c_double
        L.orc_pred_intf.argtypes = [P(C.c_double), P(C.c_double)]
        L.orc_pred_intf_batch.restype = None
        L.orc_pred_intf_batch.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_count_space.restype = C.c_uint64
        L.orc_count_space.argtypes = [C.POINTER(ProblemS), C.POINTER(Group), C.c_int64]
        L.orc_intf_loss.restype = C.c_double
        L.orc_intf_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_coll.restype = C.c_double
        L.orc_coll.argtypes = [P(ProblemS), C.c_int, C.c_double, C.c_int, C.c_int]
        L.orc_enumerate.argtypes = [P(ProblemS), P(Group), C.c_int64, P(C.c_int64), P(C.c_uint64)]
        L.orc_eval_detail.argtypes = [P(ProblemS), P(Group)] + [C.c_int] * 7 + [P(Detail)]
        L.orc_eval_indices.argtypes = [P(ProblemS), P(Group), C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_eval_range.argtypes = [P(ProblemS), P(Group), C.c_int64, C.c_uint64, C.c_uint64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_frontier_points.restype = C.c_int64
        L.orc_frontier_points.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.orc_group_frontier.argtypes = [P(ProblemS), P(Group), C.c_int64, C.c_int64, C.c_int, C.c_int,
                                         C.c_void_p, C.c_int64, P(C.c_int64), P(C.c_uint64),
                                         P(C.c_uint64)]
        L.orc_sweep.argtypes = [P(ProblemS), P(Group), C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                C.c_int, C.c_void_p, C.c_int64, P(C.c_int64), C.c_void_p,
                                C.c_void_p, C.c_void_p]
        L.orc_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, P(Group), C.c_int32, C.c_void_p,
                                 C.c_int64, P(C.c_int64), C.c_void_p]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        _lib = L
    return _lib


def _ptr(arr: np.ndarray):
    return arr.ctypes.data_as(C.c_void_p) if arr is not None else None


class Oracle:
    """Holds one synthetic problem (``synth.Problem``) in oracle form."""

    def __init__(self, pb):
        self.pb = pb
        m = pb.model
        self._keep = []
        s = ProblemS()
        s.model = Model(m.L, m.h, m.a, m.k, m.f, m.V, m.s, m.e, m.g, m.p, m.fl, m.nrm)
        s.B, s.N, s.M, s.mem_budget, s.Q = pb.B, pb.N, pb.M, pb.mem_budget, pb.Q
        s.zero_mask, s.max_stages = pb.zero_mask, pb.max_stages
        s.ckpt_ends_only = int(getattr(pb, "ckpt_ends_only", 0))
        s.offload_off = int(getattr(pb, "offload_off", 0))
        if pb.grad_accum:
            ga = np.asarray(pb.grad_accum, dtype=np.int32)
            self._keep.append(ga)
            s.n_grad_accum, s.grad_accum = len(ga), ga.ctypes.data_as(C.POINTER(C.c_int32))
        bv = np.asarray(pb.b_values, dtype=np.int32)
        tv = np.asarray(pb.tp_values, dtype=np.int32)
        self._keep += [bv, tv]
        s.n_b, s.b_values = len(bv), bv.ctypes.data_as(C.POINTER(C.c_int32))
        s.n_tp, s.tp_values = len(tv), tv.ctypes.data_as(C.POINTER(C.c_int32))
        for name in ("Tf", "Tb", "Tef", "Teb", "Thf", "Thb"):
            arr = np.ascontiguousarray(getattr(pb, name), dtype=np.float64)
            self._keep.append(arr)
            setattr(s, name, arr.ctypes.data_as(C.POINTER(C.c_double)))
        for i in range(4):
            for j in range(2):
                s.bw[i][j] = pb.bw[i][j]
                s.lat[i][j] = pb.lat[i][j]
        s.bw_h2d, s.bw_d2h = pb.bw_h2d, pb.bw_d2h
        for i in range(16):
            for j in range(4):
                s.intf[i][j] = pb.intf[i][j]
        self.s = s
        self.groups, self.n_configs = self._enumerate()

    # ---- O2/O3
    def _enumerate(self):
        L = lib()
        ng, nc = C.c_int64(0), C.c_uint64(0)
        rc = L.orc_enumerate(C.byref(self.s), None, 0, C.byref(ng), C.byref(nc))
        if rc != 0:
            raise ValueError(f"orc_enumerate failed rc={rc}")
        arr = (Group * ng.value)()
        rc = L.orc_enumerate(C.byref(self.s), arr, ng.value, C.byref(ng), C.byref(nc))
        if rc != 0:
            raise ValueError(f"orc_enumerate failed rc={rc}")
        return arr, nc.value

    @property
    def n_groups(self) -> int:
        return len(self.groups)

    def group_keys(self) -> List[Tuple[int, ...]]:
        return [(g.G, g.first, g.last, g.w, g.l, g.n, g.m) for g in self.groups]

    def group_table(self) -> np.ndarray:
        """(n_groups, 10) int64: G first last w l n m n_splits config_offset count"""
        return np.array([(g.G, g.first, g.last, g.w, g.l, g.n, g.m, g.n_splits, g.config_offset,
                          g.count) for g in self.groups], dtype=np.int64)

    def count_space(self) -> int:
        """Configurations the preset admits, counted one by one (small spaces)."""
        return int(lib().orc_count_space(C.byref(self.s), self.groups, self.n_groups))

    def n_tuples(self) -> int:
        R = (self.pb.Q + 1) ** 4
        return int(self.n_configs // R)

    # ---- O4-O9
    def detail(self, gi: int, split: int, z: int, c: int, kW: int, kG: int, kO: int, kA: int) -> Detail:
        out = Detail()
        rc = lib().orc_eval_detail(C.byref(self.s), C.byref(self.groups[gi]), split, z, c, kW, kG, kO,
                                   kA, C.byref(out))
        if rc != 0:
            raise ValueError(f"orc_eval_detail rc={rc}")
        return out

    def eval_indices(self, idx) -> Dict[str, np.ndarray]:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        n = len(idx)
        t, d, mem = (np.empty(n) for _ in range(3))
        fe = np.empty(n, dtype=np.uint8)
        rc = lib().orc_eval_indices(C.byref(self.s), self.groups, self.n_groups, _ptr(idx), n,
                                    _ptr(t), _ptr(d), _ptr(mem), _ptr(fe))
        if rc != 0:
            raise ValueError(f"orc_eval_indices rc={rc}")
        return dict(t=t, d=d, mem=mem, feasible=fe)

    def eval_range(self, begin: int, end: int) -> Dict[str, np.ndarray]:
        n = end - begin
        t, d, mem = (np.empty(n) for _ in range(3))
        fe = np.empty(n, dtype=np.uint8)
        rc = lib().orc_eval_range(C.byref(self.s), self.groups, self.n_groups, begin, end, _ptr(t),
                                  _ptr(d), _ptr(mem), _ptr(fe))
        if rc != 0:
            raise ValueError(f"orc_eval_range rc={rc}")
        return dict(t=t, d=d, mem=mem, feasible=fe)

    # ---- O10
    def group_frontier(self, g: int, ykey: int = 0, method: int = 0):
        L = lib()
        n, fc, fh = C.c_int64(0), C.c_uint64(0), C.c_uint64(0)
        cap = 1 << 16
        while True:
            out = np.zeros(cap, dtype=POINT_DTYPE)
            rc = L.orc_group_frontier(C.byref(self.s), self.groups, self.n_groups, g, ykey, method,
                                      _ptr(out), cap, C.byref(n), C.byref(fc), C.byref(fh))
            if rc == -3:
                cap *= 4
                continue
            if rc != 0:
                raise ValueError(f"orc_group_frontier rc={rc}")
            return out[: n.value].copy(), fc.value, fh.value

    def sweep(self, g_begin: int = 0, g_end: Optional[int] = None, ykey: int = 0,
              threads: Optional[int] = None):
        """Frontiers + fingerprints of groups [g_begin, g_end)."""
        L = lib()
        if g_end is None:
            g_end = self.n_groups
        if threads is None:
            threads = os.cpu_count() or 1
        ng = g_end - g_begin
        offs = np.zeros(ng + 1, dtype=np.int64)
        fc = np.zeros(ng, dtype=np.uint64)
        fh = np.zeros(ng, dtype=np.uint64)
        n = C.c_int64(0)
        cap = max(1024, ng * 64)
        while True:
            out = np.zeros(cap, dtype=POINT_DTYPE)
            rc = L.orc_sweep(C.byref(self.s), self.groups, self.n_groups, g_begin, g_end, ykey,
                             threads, _ptr(out), cap, C.byref(n), _ptr(offs), _ptr(fc), _ptr(fh))
            if rc == -3:
                cap *= 4
                continue
            if rc != 0:
                raise ValueError(f"orc_sweep rc={rc}")
            return dict(points=out[: n.value].copy(), offsets=offs, fp_count=fc, fp_hash=fh)

    def sample(self, points: np.ndarray, offsets: np.ndarray, K: int = 16,
               g_begin: int = 0) -> Tuple[np.ndarray, np.ndarray]:
        L = lib()
        ng = len(offsets) - 1
        pts = np.ascontiguousarray(points, dtype=POINT_DTYPE)
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        cap = max(1, ng * K)
        picked = np.zeros(cap, dtype=np.int64)
        poffs = np.zeros(ng + 1, dtype=np.int64)
        n = C.c_int64(0)
        grp = (Group * ng)(*[self.groups[g_begin + i] for i in range(ng)])
        rc = L.orc_sample(_ptr(pts), _ptr(offs), ng, grp, K, _ptr(picked), cap, C.byref(n), _ptr(poffs))
        if rc != 0:
            raise ValueError(f"orc_sample rc={rc}")
        return picked[: n.value].copy(), poffs


def pred_intf(X, F) -> float:
    x = (C.c_double * 4)(*X)
    f = (C.c_double * 64)(*[v for row in F for v in row])
    return lib().orc_pred_intf(x, f)


def pred_intf_batch(X: np.ndarray, F) -> np.ndarray:
    """Alg. 1 on every row of X[n][4] (literal routine, row by row)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Fa = np.ascontiguousarray(F, dtype=np.float64).reshape(16, 4)
    T = np.empty(len(X))
    lib().orc_pred_intf_batch(_ptr(X), len(X), _ptr(Fa), _ptr(T))
    return T


def intf_loss(X: np.ndarray, Tobs: np.ndarray, F) -> float:
    X = np.ascontiguousarray(X, dtype=np.float64)
    Tobs = np.ascontiguousarray(Tobs, dtype=np.float64)
    Fa = np.ascontiguousarray(F, dtype=np.float64).reshape(16, 4)
    return lib().orc_intf_loss(_ptr(X), _ptr(Tobs), len(X), _ptr(Fa))


def frontier_points(points: np.ndarray, method: int = 0) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=POINT_DTYPE)
    out = np.zeros(len(pts) + 1, dtype=POINT_DTYPE)
    n = lib().orc_frontier_points(_ptr(pts), len(pts), method, _ptr(out))
    return out[:n].copy()


def splitmix64(x: int) -> int:
    return lib().orc_splitmix64(x)
