"""Thin ctypes binding of libmist (include/mist.h).  Argument marshalling only:
every step of the sweep runs in the CUDA kernels of ``csrc/``.

The function names mirror the C ABI: ``mist_enumerate_space``,
``mist_eval_stage_costs``, ``mist_eval_stage_costs_at``,
``mist_pareto_frontier``, ``mist_sample_frontier``.  Inputs are described by
any object with the attributes of ``synth.Problem`` (model shape, B, N, M,
mem_budget, Q, zero_mask, max_stages, grad_accum and coefficient tables).

There is no CPU fallback: if ``libmist.so`` is missing this module raises on
import of the library, and without a CUDA device ``Context`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmist.so")
if os.environ.get("MIST_COUNTERS") == "1":   # instrumented build (python -m paper_2503_19050_b200.build --counters)
    LIB_PATH = os.path.join(HERE, "libmist_counters.so")
if os.environ.get("MIST_LIB"):                # A/B measurements against another build of the same ABI
    LIB_PATH = os.environ["MIST_LIB"]
MAX_SPLITS = 8
NCCL_ID_BYTES = 128

STATUS = {0: "MIST_OK", 1: "MIST_ERR_INVALID_ARG", 2: "MIST_ERR_EMPTY_SPACE",
          3: "MIST_ERR_BUFFER_TOO_SMALL", 4: "MIST_ERR_CUDA", 5: "MIST_ERR_NCCL", 6: "MIST_ERR_OOM"}
Y_DELTA, Y_MEM = 0, 1

EXPORTED = ("mist_ctx_create", "mist_ctx_destroy", "mist_status_string", "mist_ctx_last_error",
            "mist_ctx_stats", "mist_ctx_set_timing", "mist_nccl_unique_id", "mist_ctx_init_comm",
            "mist_shard_ranges",
            "mist_enumerate_space", "mist_eval_stage_costs", "mist_eval_stage_costs_at",
            "mist_pareto_frontier", "mist_frontier_points", "mist_sample_frontier",
            "mist_sample_frontier_gpu", "mist_pareto_sample", "mist_solve_inter", "mist_pred_intf", "mist_fit_intf", "mist_count_space")


class MistError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)} {detail}".strip())


class mist_model_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "num_layers", "hidden", "heads", "kv_heads", "ffn", "vocab", "seq", "elem_bytes",
        "gated_mlp", "parallel_attn", "flash_attn", "norm_vecs_per_layer")]


class mist_mesh_t(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("gpus_per_node", C.c_int32), ("mem_budget_bytes", C.c_int64)]


class mist_space_t(C.Structure):
    _fields_ = [("offload_steps", C.c_int32), ("zero_mask", C.c_int32), ("max_stages", C.c_int32),
                ("n_grad_accum", C.c_int32), ("grad_accum", C.POINTER(C.c_int32)),
                ("ckpt_ends_only", C.c_int32), ("offload_off", C.c_int32)]


class mist_coeffs_t(C.Structure):
    _fields_ = [("n_b", C.c_int32), ("b_values", C.POINTER(C.c_int32)),
                ("n_tp", C.c_int32), ("tp_values", C.POINTER(C.c_int32))] + [
        (n, C.POINTER(C.c_double)) for n in ("t_layer_fwd", "t_layer_bwd", "t_emb_fwd", "t_emb_bwd",
                                              "t_head_fwd", "t_head_bwd")] + [
        ("bw", (C.c_double * 2) * 4), ("lat", (C.c_double * 2) * 4),
        ("bw_h2d", C.c_double), ("bw_d2h", C.c_double), ("intf", (C.c_double * 4) * 16)]


class mist_group_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("G", "first", "last", "w", "layers", "n", "m", "n_splits")] + [
        ("tp", C.c_int32 * MAX_SPLITS), ("dp", C.c_int32 * MAX_SPLITS), ("b", C.c_int32 * MAX_SPLITS),
        ("tuple_offset", C.c_uint64), ("config_offset", C.c_uint64), ("count", C.c_uint64)]


class mist_point_t(C.Structure):
    _fields_ = [("idx", C.c_uint64), ("t", C.c_double), ("y", C.c_double), ("mem", C.c_double)]


class mist_stats_t(C.Structure):
    _fields_ = [("configs_evaluated", C.c_uint64), ("candidates", C.c_uint64),
                ("frontier_points", C.c_uint64), ("kernel_launches", C.c_int64),
                ("eval_ms", C.c_double), ("precompute_ms", C.c_double), ("reduce_ms", C.c_double),
                ("merge_ms", C.c_double), ("total_ms", C.c_double), ("chunks", C.c_int64),
                ("reductions", C.c_int64), ("sort_keys", C.c_uint64), ("sort_passes", C.c_int32),
                ("unit_factors", C.c_int32), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("pilot_ms", C.c_double), ("pilot_configs", C.c_uint64), ("rollbacks", C.c_int64),
                ("phases_evaluated", C.c_uint64), ("bound_rows", C.c_uint64)]


MAX_STAGES = 128


class mist_plan_t(C.Structure):
    _fields_ = [("G", C.c_int32), ("S", C.c_int32), ("objective", C.c_double), ("t_max", C.c_double),
                ("t_sum", C.c_double), ("d_term", C.c_double), ("labels", C.c_int64),
                ("group", C.c_int32 * MAX_STAGES), ("point", C.c_int64 * MAX_STAGES)]


POINT_DTYPE = np.dtype([("idx", "<u8"), ("t", "<f8"), ("y", "<f8"), ("mem", "<f8")])
assert POINT_DTYPE.itemsize == C.sizeof(mist_point_t) == 32

_lib = None


def lib():
    """Load libmist.so (built in-tree by ``paper_2503_19050_b200.build``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libmist.so not built ({LIB_PATH}); run python -m paper_2503_19050_b200.build")
        L = C.CDLL(LIB_PATH)
        P, V = C.POINTER, C.c_void_p
        L.mist_status_string.restype = C.c_char_p
        L.mist_ctx_last_error.restype = C.c_char_p
        L.mist_ctx_last_error.argtypes = [V]
        L.mist_ctx_create.argtypes = [C.c_int, P(V)]
        L.mist_ctx_destroy.argtypes = [V]
        L.mist_ctx_destroy.restype = None
        L.mist_ctx_stats.argtypes = [V, P(mist_stats_t)]
        L.mist_ctx_set_timing.argtypes = [V, C.c_int]
        L.mist_nccl_unique_id.argtypes = [V]
        L.mist_ctx_init_comm.argtypes = [V, V, C.c_int, C.c_int]
        L.mist_shard_ranges.argtypes = [C.c_uint64, C.c_int, C.c_int, V, V, C.c_int64, P(C.c_int64)]
        L.mist_enumerate_space.argtypes = [P(mist_model_t), C.c_int64, P(mist_mesh_t), P(mist_space_t),
                                           P(mist_coeffs_t), P(mist_group_t), C.c_int64, P(C.c_int64),
                                           P(C.c_uint64)]
        common = [V, P(mist_model_t), C.c_int64, P(mist_mesh_t), P(mist_space_t), P(mist_coeffs_t),
                  P(mist_group_t), C.c_int64]
        L.mist_eval_stage_costs.argtypes = common + [C.c_uint64, C.c_uint64, V, V, V, V]
        L.mist_eval_stage_costs_at.argtypes = common + [V, C.c_int64, V, V, V, V]
        if hasattr(L, "mist_pareto_sample") or not os.environ.get("MIST_LIB"):   # older A/B builds lack a12-dev
            L.mist_sample_frontier_gpu.argtypes = [V, V, C.c_int64, V, C.c_int64, P(mist_group_t), C.c_int32, V, V]
            L.mist_pareto_sample.argtypes = common + [C.c_uint64, C.c_uint64, C.c_int32, V, V]
        L.mist_pareto_frontier.argtypes = common + [C.c_uint64, C.c_uint64, C.c_int, V, C.c_int64,
                                                    P(C.c_int64), V, V, V]
        L.mist_sample_frontier.argtypes = [V, V, C.c_int64, P(mist_group_t), C.c_int32, V, C.c_int64,
                                           P(C.c_int64), V]
        L.mist_frontier_points.argtypes = [V, V, V, C.c_int64, C.c_int64, V, C.c_int64, P(C.c_int64), V]
        if hasattr(L, "mist_count_space"):
            L.mist_count_space.argtypes = [P(mist_model_t), C.c_int64, P(mist_mesh_t), P(mist_space_t),
                                           P(C.c_uint64), P(C.c_uint64)]
        if hasattr(L, "mist_fit_intf"):
            L.mist_pred_intf.argtypes = [V, V, C.c_int64, V, V]
            L.mist_fit_intf.argtypes = [V, V, V, C.c_int64, V, C.c_int32, C.c_double, V, P(C.c_double)]
        if hasattr(L, "mist_solve_inter"):
            L.mist_solve_inter.argtypes = [V, C.c_int64, V, V, C.c_int32, C.c_int32, C.c_int32, P(mist_plan_t)]
        for name in EXPORTED:
            if name not in ("mist_ctx_destroy", "mist_status_string", "mist_ctx_last_error"):
                if os.environ.get("MIST_LIB") and not hasattr(L, name):
                    continue
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _ptr(x) -> Optional[int]:
    """Raw address of a numpy array or a torch tensor (None passes NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, int):
        return x
    raise TypeError(type(x))


class Spec:
    """The C structs of one problem, kept alive together."""

    def __init__(self, pb):
        m = pb.model
        self._keep = []
        self.model = mist_model_t(m.L, m.h, m.a, m.k, m.f, m.V, m.s, m.e, m.g, m.p, m.fl, m.nrm)
        self.B = int(pb.B)
        self.mesh = mist_mesh_t(pb.N, pb.M, int(pb.mem_budget))
        self.space = mist_space_t(pb.Q, pb.zero_mask, pb.max_stages, 0, None,
                                  int(getattr(pb, "ckpt_ends_only", 0)), int(getattr(pb, "offload_off", 0)))
        if pb.grad_accum:
            ga = np.ascontiguousarray(pb.grad_accum, dtype=np.int32)
            self._keep.append(ga)
            self.space.n_grad_accum = len(ga)
            self.space.grad_accum = ga.ctypes.data_as(C.POINTER(C.c_int32))
        c = mist_coeffs_t()
        bv = np.ascontiguousarray(pb.b_values, dtype=np.int32)
        tv = np.ascontiguousarray(pb.tp_values, dtype=np.int32)
        self._keep += [bv, tv]
        c.n_b, c.b_values = len(bv), bv.ctypes.data_as(C.POINTER(C.c_int32))
        c.n_tp, c.tp_values = len(tv), tv.ctypes.data_as(C.POINTER(C.c_int32))
        for cname, pname in (("t_layer_fwd", "Tf"), ("t_layer_bwd", "Tb"), ("t_emb_fwd", "Tef"),
                             ("t_emb_bwd", "Teb"), ("t_head_fwd", "Thf"), ("t_head_bwd", "Thb")):
            arr = np.ascontiguousarray(getattr(pb, pname), dtype=np.float64)
            self._keep.append(arr)
            setattr(c, cname, arr.ctypes.data_as(C.POINTER(C.c_double)))
        for i in range(4):
            for j in range(2):
                c.bw[i][j] = pb.bw[i][j]
                c.lat[i][j] = pb.lat[i][j]
        c.bw_h2d, c.bw_d2h = pb.bw_h2d, pb.bw_d2h
        for i in range(16):
            for j in range(4):
                c.intf[i][j] = pb.intf[i][j]
        self.coeffs = c
        self.groups, self.n_configs = mist_enumerate_space(self)
        self.n_groups = len(self.groups)
        Q1 = pb.Q + 1
        self.R = Q1 ** 4
        self.n_tuples = self.n_configs // self.R

    def args(self):
        return (C.byref(self.model), self.B, C.byref(self.mesh), C.byref(self.space),
                C.byref(self.coeffs), self.groups, self.n_groups)


def mist_enumerate_space(spec: Spec, with_coeffs: bool = True):
    L = lib()
    ng, nc = C.c_int64(0), C.c_uint64(0)
    cf = C.byref(spec.coeffs) if with_coeffs else None
    st = L.mist_enumerate_space(C.byref(spec.model), spec.B, C.byref(spec.mesh), C.byref(spec.space), cf,
                                None, 0, C.byref(ng), C.byref(nc))
    if st != 0:
        raise MistError(st, "mist_enumerate_space")
    groups = (mist_group_t * ng.value)()
    st = L.mist_enumerate_space(C.byref(spec.model), spec.B, C.byref(spec.mesh), C.byref(spec.space), cf,
                                groups, ng.value, C.byref(ng), C.byref(nc))
    if st != 0:
        raise MistError(st, "mist_enumerate_space")
    return groups, nc.value


class Context:
    """One device context (stream, scratch, optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        st = lib().mist_ctx_create(device, C.byref(self._h))
        if st != 0:
            raise MistError(st, "mist_ctx_create", "(no usable CUDA device?)")
        self.device = device

    def close(self):
        if self._h:
            lib().mist_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def last_error(self) -> str:
        return lib().mist_ctx_last_error(self._h).decode()

    def check(self, st: int, where: str):
        if st != 0:
            raise MistError(st, where, self.last_error())

    def stats(self) -> dict:
        s = mist_stats_t()
        self.check(lib().mist_ctx_stats(self._h, C.byref(s)), "mist_ctx_stats")
        return {name: getattr(s, name) for name, _ in mist_stats_t._fields_}

    def set_timing(self, enabled: bool):
        self.check(lib().mist_ctx_set_timing(self._h, int(enabled)), "mist_ctx_set_timing")

    def init_comm(self, nccl_id: bytes, rank: int, world: int):
        buf = (C.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(nccl_id)
        self.check(lib().mist_ctx_init_comm(self._h, buf, rank, world), "mist_ctx_init_comm")


def mist_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * NCCL_ID_BYTES)()
    st = lib().mist_nccl_unique_id(buf)
    if st != 0:
        raise MistError(st, "mist_nccl_unique_id")
    return bytes(buf)


def mist_shard_ranges(n_tuples: int, rank: int, world: int) -> List[Tuple[int, int]]:
    """This rank's block-cyclic share of the tuple range, as [begin, end) pairs (host-only)."""
    n = C.c_int64(0)
    st = lib().mist_shard_ranges(n_tuples, rank, world, None, None, 0, C.byref(n))
    if st != 0:
        raise MistError(st, "mist_shard_ranges")
    b = (C.c_uint64 * max(1, n.value))()
    e = (C.c_uint64 * max(1, n.value))()
    st = lib().mist_shard_ranges(n_tuples, rank, world, b, e, n.value, C.byref(n))
    if st != 0:
        raise MistError(st, "mist_shard_ranges")
    return [(b[i], e[i]) for i in range(n.value)]


def mist_eval_stage_costs(ctx: Context, spec: Spec, begin: int, end: int, t=None, d=None, mem=None,
                          feasible=None):
    """Dense evaluation of [begin, end); outputs are CUDA tensors (or None)."""
    st = lib().mist_eval_stage_costs(ctx.handle, *spec.args(), begin, end, _ptr(t), _ptr(d), _ptr(mem),
                                     _ptr(feasible))
    ctx.check(st, "mist_eval_stage_costs")


def mist_eval_stage_costs_at(ctx: Context, spec: Spec, idx, t=None, d=None, mem=None, feasible=None):
    """idx: CUDA uint64/int64 tensor of global config indices."""
    st = lib().mist_eval_stage_costs_at(ctx.handle, *spec.args(), _ptr(idx), int(idx.numel()), _ptr(t),
                                        _ptr(d), _ptr(mem), _ptr(feasible))
    ctx.check(st, "mist_eval_stage_costs_at")


def mist_pareto_frontier(ctx: Context, spec: Spec, t_begin: int = 0, t_end: int = 0, ykey: int = Y_DELTA,
                         fingerprints: bool = False, out=None, group_offsets=None):
    """Returns (points[np structured POINT_DTYPE], group_offsets[int64], fp_count, fp_hash).

    ``out`` / ``group_offsets`` may be caller-provided host arrays or device
    tensors; by default host numpy arrays are allocated (two-call pattern on
    BUFFER_TOO_SMALL)."""
    L = lib()
    ng = spec.n_groups
    n = C.c_int64(0)
    offs = group_offsets if group_offsets is not None else np.zeros(ng + 1, dtype=np.int64)
    fpc = np.zeros(ng, dtype=np.uint64) if fingerprints else None
    fph = np.zeros(ng, dtype=np.uint64) if fingerprints else None
    if out is None:
        cap = max(1024, 64 * ng)
        pts = np.empty(cap, dtype=POINT_DTYPE)     # written by the library up to n_out
    else:
        pts = out
        cap = len(out) if isinstance(out, np.ndarray) else out.numel() // 4
    st = L.mist_pareto_frontier(ctx.handle, *spec.args(), t_begin, t_end, ykey, _ptr(pts), cap, C.byref(n),
                                _ptr(offs), _ptr(fpc), _ptr(fph))
    if st == 3 and out is None:
        pts = np.empty(n.value, dtype=POINT_DTYPE)
        st = L.mist_pareto_frontier(ctx.handle, *spec.args(), t_begin, t_end, ykey, _ptr(pts), n.value,
                                    C.byref(n), _ptr(offs), _ptr(fpc), _ptr(fph))
    ctx.check(st, "mist_pareto_frontier")
    if isinstance(pts, np.ndarray):
        pts = pts[: n.value]
    return pts, offs, fpc, fph


def mist_frontier_points(ctx: Context, points, groups, n_groups: int, out=None, group_offsets=None):
    """Exact per-group frontier of an explicit point set (O12 merge).

    points: POINT_DTYPE numpy array or a CUDA tensor holding n*4 float64/int64
    words; groups: int32 numpy array or CUDA tensor.  Returns (points, offsets)."""
    L = lib()
    n = len(points) if isinstance(points, np.ndarray) else points.numel() // 4
    offs = group_offsets if group_offsets is not None else np.zeros(n_groups + 1, dtype=np.int64)
    cap = n if out is None else (len(out) if isinstance(out, np.ndarray) else out.numel() // 4)
    res = np.zeros(max(1, cap), dtype=POINT_DTYPE) if out is None else out
    m = C.c_int64(0)
    st = L.mist_frontier_points(ctx.handle, _ptr(points), _ptr(groups), n, n_groups, _ptr(res), cap,
                                C.byref(m), _ptr(offs))
    ctx.check(st, "mist_frontier_points")
    if isinstance(res, np.ndarray):
        res = res[: m.value]
    return res, offs


def mist_sample_frontier(points: np.ndarray, offsets: np.ndarray, spec: Spec, K: int = 16
                         ) -> Tuple[np.ndarray, np.ndarray]:
    L = lib()
    ng = len(offsets) - 1
    pts = np.ascontiguousarray(points, dtype=POINT_DTYPE)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    cap = max(1, ng * K)
    picked = np.zeros(cap, dtype=np.int64)
    poffs = np.zeros(ng + 1, dtype=np.int64)
    n = C.c_int64(0)
    st = L.mist_sample_frontier(_ptr(pts), _ptr(offs), ng, spec.groups, K, _ptr(picked), cap, C.byref(n),
                                _ptr(poffs))
    if st != 0:
        raise MistError(st, "mist_sample_frontier")
    return picked[: n.value], poffs


def mist_sample_frontier_gpu(ctx: Context, points, offsets, spec: Spec, K: int = 16):
    """a12 on the device.  points/offsets: numpy (POINT_DTYPE / int64) or CUDA
    tensors.  Returns (picked[n_groups, K] int64 positions, -1 padded;
    n_picked[n_groups] int32) as numpy arrays."""
    ng = spec.n_groups
    if isinstance(points, np.ndarray):
        points = np.ascontiguousarray(points, dtype=POINT_DTYPE)
        npts = len(points)
    else:
        npts = points.numel() // 4
    if isinstance(offsets, np.ndarray):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    picked = np.zeros((ng, K), dtype=np.int64)
    npk = np.zeros(ng, dtype=np.int32)
    st = lib().mist_sample_frontier_gpu(ctx.handle, _ptr(points), npts, _ptr(offsets), ng, spec.groups, K,
                                        _ptr(picked), _ptr(npk))
    ctx.check(st, "mist_sample_frontier_gpu")
    return picked, npk


def mist_pareto_sample(ctx: Context, spec: Spec, K: int = 16, t_begin: int = 0, t_end: int = 0):
    """Sweep + device a12: returns (samples[n_groups, K] POINT_DTYPE, n_picked[n_groups])."""
    ng = spec.n_groups
    out = np.zeros(ng * K, dtype=POINT_DTYPE)
    npk = np.zeros(ng, dtype=np.int32)
    st = lib().mist_pareto_sample(ctx.handle, *spec.args(), t_begin, t_end, K, _ptr(out), _ptr(npk))
    ctx.check(st, "mist_pareto_sample")
    return out.reshape(ng, K), npk


def group_array(keys) -> "C.Array":
    """mist_group_t[] holding only the keys (G, first, last, w, l, n, m): the
    part of the group table that mist_solve_inter reads."""
    arr = (mist_group_t * len(keys))()
    for i, k in enumerate(keys):
        g = arr[i]
        g.G, g.first, g.last, g.w, g.layers, g.n, g.m = (int(v) for v in k)
    return arr


def mist_solve_inter(groups, points: np.ndarray, offsets: np.ndarray, num_layers: int, n_devices: int,
                     n_threads: int = 0) -> dict:
    """Inter-stage plan (Eq. 2-3) over per-group candidates (CSR: points, offsets).
    groups: a ctypes mist_group_t array (``Spec.groups`` or ``group_array``).
    Returns dict(G, S, objective, t_max, t_sum, d_term, labels, group[S], point[S])."""
    if points.dtype != POINT_DTYPE:            # e.g. records carrying extra fields
        pts = np.zeros(len(points), dtype=POINT_DTYPE)
        for f in POINT_DTYPE.names:
            pts[f] = points[f]
    else:
        pts = np.ascontiguousarray(points)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    plan = mist_plan_t()
    st = lib().mist_solve_inter(C.addressof(groups), len(groups), _ptr(pts) if len(pts) else None, _ptr(offs),
                                int(num_layers), int(n_devices), int(n_threads), C.byref(plan))
    if st != 0:
        raise MistError(st, "mist_solve_inter")
    S = plan.S
    return dict(G=plan.G, S=S, objective=plan.objective, t_max=plan.t_max, t_sum=plan.t_sum,
                d_term=plan.d_term, labels=plan.labels, group=np.array(plan.group[:S], dtype=np.int64),
                point=np.array(plan.point[:S], dtype=np.int64))


def _table(F) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(16, 4))


def mist_pred_intf(ctx: Context, X, F, T=None):
    """Alg. 1 on every row of X (CUDA tensor [n, 4] float64).  Returns T (CUDA tensor [n])."""
    import torch
    n = X.shape[0]
    if T is None:
        T = torch.empty(n, dtype=torch.float64, device=X.device)
    tab = _table(F)
    st = lib().mist_pred_intf(ctx.handle, _ptr(X), n, _ptr(tab), _ptr(T))
    ctx.check(st, "mist_pred_intf")
    return T


def mist_fit_intf(ctx: Context, X, T_obs, init, iters: int = 2, fmax: float = 4.0):
    """Fit the 28 member factors to observations (CUDA tensors X [n, 4], T_obs [n]).
    Returns (table[16, 4] numpy, loss)."""
    tab = _table(init)
    out = np.zeros((16, 4), dtype=np.float64)
    loss = C.c_double(0.0)
    st = lib().mist_fit_intf(ctx.handle, _ptr(X), _ptr(T_obs), X.shape[0], _ptr(tab), int(iters), float(fmax),
                             _ptr(out), C.byref(loss))
    ctx.check(st, "mist_fit_intf")
    return out, loss.value


def mist_count_space(spec: Spec) -> Tuple[int, int]:
    """(configurations the preset admits, size of the full index space)."""
    a, b = C.c_uint64(0), C.c_uint64(0)
    st = lib().mist_count_space(C.byref(spec.model), spec.B, C.byref(spec.mesh), C.byref(spec.space),
                                C.byref(a), C.byref(b))
    if st != 0:
        raise MistError(st, "mist_count_space")
    return a.value, b.value
