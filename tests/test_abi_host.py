"""CPU-side checks of the C ABI (no GPU): the library loads, exports every
symbol include/mist.h declares, its host-only entry points (a1 enumeration,
a12 sampling) agree with the oracle bit for bit, and argument errors map to
the documented status codes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.binding import Oracle
from paper_2503_19050_b200 import build as mist_build
from paper_2503_19050_b200 import mist
from synth import random_problem, tiny, workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    mist_build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mist.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(mist_[a-z_0-9]+)\s*\(", hdr))
    assert {"mist_enumerate_space", "mist_eval_stage_costs", "mist_pareto_frontier",
            "mist_sample_frontier"} <= declared
    L = C.CDLL(mist.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(mist.EXPORTED)


def test_library_is_sm100a():
    """The fatbin holds sm_100a SASS (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", mist.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _keys(groups, layers_field="layers"):
    return [(g.G, g.first, g.last, g.w, getattr(g, layers_field), g.n, g.m, g.n_splits,
             tuple(g.tp[:g.n_splits]), tuple(g.dp[:g.n_splits]), tuple(g.b[:g.n_splits]),
             g.tuple_offset, g.config_offset, g.count) for g in groups]


@pytest.mark.parametrize("which", ["tiny1", "tiny2", "tiny3", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
                         + [f"rand{i}" for i in range(12)])
def test_enumeration_bit_exact_vs_oracle(which):
    if which.startswith("tiny"):
        pb = {"tiny1": tiny(2, 2, 1, 2, 2, 1), "tiny2": tiny(2, 2, 1, 2, 4, 2),
              "tiny3": tiny(5, 4, 2, 4, 12, 2)}[which]
    elif which.startswith("cfg"):
        pb = workload(int(which[3:]))
    else:
        pb = random_problem(int(which[4:]))
    try:
        o = Oracle(pb)
    except ValueError:
        with pytest.raises(mist.MistError) as ei:
            mist.Spec(pb)
        assert ei.value.status == 2   # EMPTY_SPACE
        return
    s = mist.Spec(pb)
    assert s.n_configs == o.n_configs
    assert _keys(s.groups) == _keys(o.groups, "l")


def test_enumeration_errors():
    pb = tiny(2, 2, 1, 2, 2, 1)
    s = mist.Spec(pb)
    L = mist.lib()
    ng, nc = C.c_int64(0), C.c_uint64(0)

    def call(**over):
        model = mist.mist_model_t.from_buffer_copy(s.model)
        mesh = mist.mist_mesh_t.from_buffer_copy(s.mesh)
        space = mist.mist_space_t.from_buffer_copy(s.space)
        B = over.pop("B", s.B)
        for k, v in over.items():
            for obj in (model, mesh, space):
                if hasattr(obj, k):
                    setattr(obj, k, v)
        return L.mist_enumerate_space(C.byref(model), B, C.byref(mesh), C.byref(space), C.byref(s.coeffs),
                                      None, 0, C.byref(ng), C.byref(nc))

    assert call() == 0
    assert call(B=0) == 1
    assert call(offload_steps=0) == 1
    assert call(zero_mask=0) == 1
    assert call(mem_budget_bytes=0) == 1
    assert call(heads=3) == 1            # a does not divide k*h... k=2,h=64: 128 % 3 != 0
    # a b value missing from the coefficient tables
    bad = mist.mist_coeffs_t.from_buffer_copy(s.coeffs)
    bv = np.array([7], dtype=np.int32)
    bad.n_b, bad.b_values = 1, bv.ctypes.data_as(C.POINTER(C.c_int32))
    assert L.mist_enumerate_space(C.byref(s.model), s.B, C.byref(s.mesh), C.byref(s.space), C.byref(bad),
                                  None, 0, C.byref(ng), C.byref(nc)) == 1
    # buffer too small
    g1 = (mist.mist_group_t * 2)()
    assert L.mist_enumerate_space(C.byref(s.model), s.B, C.byref(s.mesh), C.byref(s.space), C.byref(s.coeffs),
                                  g1, 2, C.byref(ng), C.byref(nc)) == 3
    assert ng.value == 6


def test_empty_space():
    """no valid (DP, TP) split anywhere -> EMPTY_SPACE.  B=3 on a 1x2
    mesh of a 2-head model: every G*DP must divide 3 but the single stage on
    2 GPUs has DP in {1 (TP=2), 2}; use heads=1 so TP=2 is impossible."""
    pb = tiny(1, 1, 1, 2, 3, 1)
    with pytest.raises(mist.MistError) as ei:
        mist.Spec(pb)
    assert ei.value.status == 2


def test_ctx_create_fails_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(mist.MistError) as ei:
        mist.Context(0)
    assert ei.value.status == 4


def test_sampling_matches_oracle():
    """a12 is host C++ in libmist: same picks as the oracle's O11 on the
    oracle's frontier."""
    for pb in (tiny(2, 2, 1, 2, 4, 2), tiny(3, 4, 1, 4, 8, 1)):
        o = Oracle(pb)
        s = mist.Spec(pb)
        res = o.sweep(threads=2)
        pts = np.zeros(len(res["points"]), dtype=mist.POINT_DTYPE)
        for f in ("idx", "t", "y", "mem"):
            pts[f] = res["points"][f]
        for K in (2, 3, 16):
            a, ao = o.sample(res["points"], res["offsets"], K=K)
            b, bo = mist.mist_sample_frontier(pts, res["offsets"], s, K=K)
            assert a.tolist() == b.tolist() and ao.tolist() == bo.tolist()
        with pytest.raises(mist.MistError):
            mist.mist_sample_frontier(pts, res["offsets"], s, K=1)
