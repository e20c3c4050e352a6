"""Seeded synthetic inputs for the intra-stage tuning sweep.

This module is the ONLY code shared by the oracle side (``oracle/``) and the
CUDA side (``paper_2503_19050_b200``).  It holds none of the method's
arithmetic (no enumeration, no cost expression, no interference model, no
memory model, no frontier): it only writes down *inputs* -- model shapes,
meshes, budgets, search-space options and the synthetic "profiled" operator
time tables that stand in for Mist's operator database (PAPER.md line 541,
Sec. 5.2.1 "operator computation database").

Recipe (SURVEY.md Sec. 8(d) "Coefficient tables"):

* Workload shapes follow the paper's Table 4 and the
  hardware profiles follow Table 3.
* Seed 250319050, ``numpy.random.Generator(PCG64(seed))``; draws in order of
  ``b`` ascending then ``tp`` in (1, 2, 4, 8), two standard normals each.
* ``flops_f = (2 b s (P_dense) + 4 b s^2 h) / tp`` where ``P_dense`` is the
  matmul weight count of one transformer layer, ``u = b s h / tp``,
  ``eff = 0.70 u / (u + 2^22)``, ``Tf = flops_f / (peak eff) (1 + 0.03 N1)``,
  ``Tb = 2 Tf (1 + 0.03 N2)``; embedding ``Tef = e b s h / 3e11``, ``Teb = 2 Tef``;
  LM head ``Thf = 2 b s h V / tp / (peak eff)``, ``Thb = 2 Thf``.
* Interference factor tables: ``unit`` (all 1, i.e. "max over streams"),
  ``spec`` (pairs 1.15, triples 1.25, quadruple 1.35) and
  ``asym`` (every member factor drawn uniformly from [1, 2], seeded) -- the
  last one exists so that a transposed channel index cannot hide behind a
  symmetric table.

Everything here is plain Python/numpy and deterministic.
"""
from __future__ import annotations

import copy
import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

SEED = 250319050

# Channel bit order of the factor table: C=1, NCCL(G2G)=2, H2D(C2G)=4, D2H(G2C)=8
# (Alg. 1 stacks X = [C, G2G, C2G, G2C]; SURVEY ledger L6).
N_CHANNELS = 4

# Hardware profiles (Table 3).
PROFILES = {
    "L4": dict(peak=121e12, capacity=24e9, h2d=12e9, d2h=12e9,
               bw_intra=8e9, bw_inter=4e9, lat=30e-6),
    "A100": dict(peak=312e12, capacity=40e9, h2d=20e9, d2h=20e9,
                 bw_intra=150e9, bw_inter=40e9, lat=20e-6),
}


@dataclasses.dataclass
class Model:
    L: int          # num_layers
    h: int          # hidden
    a: int          # heads
    k: int          # kv heads
    f: int          # ffn
    V: int          # vocab
    s: int          # sequence length
    e: int = 2      # bytes per element (FP16 mixed precision)
    g: int = 0      # gated MLP
    p: int = 0      # parallel attention
    fl: int = 1     # flash attention
    nrm: int = 4    # norm weight vectors per layer


@dataclasses.dataclass
class Problem:
    name: str
    model: Model
    B: int                      # global batch
    N: int                      # nodes
    M: int                      # gpus per node
    mem_budget: int             # bytes per GPU
    Q: int                      # offload ratio steps (ratio grid k/Q)
    zero_mask: int = 0xF        # allowed ZeRO levels (bit z)
    max_stages: int = 0         # 0 => min(L, N*M)
    ckpt_ends_only: int = 0     # preset: CKPT c in {0, l} only
    offload_off: int = 0        # preset: bit 0 WO, 1 GO, 2 OO, 3 AO fixed at 0
    grad_accum: Optional[List[int]] = None   # None => all divisors of B
    profile: str = "L4"
    factors: str = "spec"       # unit | spec | asym
    # coefficient tables (filled by make_coeffs)
    b_values: List[int] = dataclasses.field(default_factory=list)
    tp_values: List[int] = dataclasses.field(default_factory=list)
    Tf: List[float] = dataclasses.field(default_factory=list)
    Tb: List[float] = dataclasses.field(default_factory=list)
    Tef: List[float] = dataclasses.field(default_factory=list)
    Teb: List[float] = dataclasses.field(default_factory=list)
    Thf: List[float] = dataclasses.field(default_factory=list)
    Thb: List[float] = dataclasses.field(default_factory=list)
    bw: List[List[float]] = dataclasses.field(default_factory=list)    # [AR,AG,RS,P2P][intra,inter]
    lat: List[List[float]] = dataclasses.field(default_factory=list)
    bw_h2d: float = 0.0
    bw_d2h: float = 0.0
    intf: List[List[float]] = dataclasses.field(default_factory=list)  # [16][4]

    def with_factors(self, name: str, seed: int = SEED) -> "Problem":
        q = copy.deepcopy(self)
        q.factors = name
        q.intf = factor_table(name, seed)
        return q

    def replace(self, **kw) -> "Problem":
        q = copy.deepcopy(self)
        for key, val in kw.items():
            setattr(q, key, val)
        return q


def divisors(x: int) -> List[int]:
    return [d for d in range(1, x + 1) if x % d == 0]


def _subsets_ge2() -> List[int]:
    return [mask for mask in range(16) if bin(mask).count("1") >= 2]


def factor_table(name: str, seed: int = SEED) -> List[List[float]]:
    """16x4 table F[mask][j]: slowdown factor of channel j when exactly the
    channels in ``mask`` run concurrently ("each possible
    combination of co-running kernels is assigned a set of slowdown factors").
    Rows with fewer than two channels are never read and are set to 1."""
    table = [[1.0] * N_CHANNELS for _ in range(16)]
    if name == "unit":
        return table
    if name == "spec":
        by_size = {2: 1.15, 3: 1.25, 4: 1.35}
        for mask in _subsets_ge2():
            n = bin(mask).count("1")
            for j in range(N_CHANNELS):
                if mask >> j & 1:
                    table[mask][j] = by_size[n]
        return table
    if name == "asym":
        rng = np.random.Generator(np.random.PCG64(seed + 7))
        for mask in _subsets_ge2():
            for j in range(N_CHANNELS):
                if mask >> j & 1:
                    table[mask][j] = float(rng.uniform(1.0, 2.0))
        return table
    raise ValueError(f"unknown factor table {name!r}")


def make_coeffs(pb: Problem, tp_values=(1, 2, 4, 8), seed: int = SEED) -> Problem:
    """Fill the synthetic operator-time tables (stand-in for the paper's
    profiled operator database) and the link tables."""
    m = pb.model
    prof = PROFILES[pb.profile]
    peak = prof["peak"]
    rng = np.random.Generator(np.random.PCG64(seed))
    b_values = divisors(pb.B)
    kvd = m.k * m.h // m.a
    # matmul weights of one layer (attention q,o + k,v + MLP): the FLOP-bearing part
    p_dense = 2 * m.h * m.h + 2 * m.h * kvd + (2 + m.g) * m.h * m.f
    Tf, Tb, Tef, Teb, Thf, Thb = [], [], [], [], [], []
    for b in b_values:
        for tp in tp_values:
            n1, n2 = rng.standard_normal(2)
            flops_f = (2.0 * b * m.s * p_dense + 4.0 * b * m.s * m.s * m.h) / tp
            u = b * m.s * m.h / tp
            eff = 0.70 * u / (u + 2.0 ** 22)
            tf = flops_f / (peak * eff) * (1.0 + 0.03 * n1)
            tb = 2.0 * tf * (1.0 + 0.03 * n2)
            tef = m.e * b * m.s * m.h / 3e11
            thf = 2.0 * b * m.s * m.h * m.V / tp / (peak * eff)
            Tf.append(float(tf)); Tb.append(float(tb))
            Tef.append(float(tef)); Teb.append(float(2.0 * tef))
            Thf.append(float(thf)); Thb.append(float(2.0 * thf))
    q = copy.deepcopy(pb)
    q.b_values = list(b_values)
    q.tp_values = list(tp_values)
    q.Tf, q.Tb, q.Tef, q.Teb, q.Thf, q.Thb = Tf, Tb, Tef, Teb, Thf, Thb
    bw = [[prof["bw_intra"], prof["bw_inter"]] for _ in range(4)]
    lat = [[prof["lat"], prof["lat"]] for _ in range(4)]
    q.bw, q.lat = bw, lat
    q.bw_h2d, q.bw_d2h = prof["h2d"], prof["d2h"]
    q.intf = factor_table(pb.factors, seed)
    return q


def budget(profile: str) -> int:
    """Mem_Budget = floor(0.9 * capacity) (SURVEY ledger L22)."""
    return int(math.floor(0.9 * PROFILES[profile]["capacity"]))


# --- the five BASELINE.json workloads -------------

GPT3_1_3B = Model(L=24, h=2048, a=16, k=16, f=8192, V=50257, s=2048, g=0, p=0, nrm=4)
GPT3_2_7B = Model(L=32, h=2560, a=32, k=32, f=10240, V=50257, s=2048, g=0, p=0, nrm=4)
LLAMA2_7B = Model(L=32, h=4096, a=32, k=32, f=11008, V=32000, s=4096, g=1, p=0, nrm=2)
GPT3_22B = Model(L=48, h=6144, a=48, k=48, f=24576, V=50257, s=2048, g=0, p=0, nrm=4)
FALCON_40B = Model(L=60, h=8192, a=128, k=8, f=32768, V=65024, s=2048, g=0, p=1, nrm=4)


def workload(i: int, factors: str = "spec") -> Problem:
    """BASELINE.json ``configs[i-1]`` (SURVEY numbering cfg1..cfg5)."""
    table = {
        1: ("cfg1_gpt3_1.3b", GPT3_1_3B, 32, 1, 4, 4, "L4"),
        2: ("cfg2_gpt3_2.7b", GPT3_2_7B, 64, 1, 8, 10, "L4"),
        3: ("cfg3_llama2_7b", LLAMA2_7B, 128, 2, 8, 20, "A100"),
        4: ("cfg4_gpt3_22b", GPT3_22B, 512, 4, 8, 8, "L4"),
        5: ("cfg5_falcon_40b", FALCON_40B, 1024, 8, 8, 50, "A100"),
    }
    name, model, B, N, M, Q, prof = table[i]
    pb = Problem(name=name, model=copy.deepcopy(model), B=B, N=N, M=M,
                 mem_budget=budget(prof), Q=Q, profile=prof, factors=factors)
    return make_coeffs(pb)


def tiny(L: int, heads: int, N: int, M: int, B: int, Q: int,
         mem_budget: int = 2_000_000, factors: str = "asym", h: int = 64,
         s: int = 128, V: int = 512, profile: str = "L4",
         kv_heads: Optional[int] = None, g: int = 0, p: int = 0, fl: int = 1) -> Problem:
    """Small synthetic shapes ("synthetic shapes with the given L,
    heads = kv heads") for brute-force and element-wise parity tests."""
    model = Model(L=L, h=h, a=heads, k=kv_heads if kv_heads else heads, f=4 * h,
                  V=V, s=s, g=g, p=p, fl=fl, nrm=4)
    pb = Problem(name=f"tiny_L{L}_a{heads}_{N}x{M}_B{B}_Q{Q}", model=model, B=B,
                 N=N, M=M, mem_budget=mem_budget, Q=Q, profile=profile,
                 factors=factors)
    return make_coeffs(pb)


def random_problem(seed: int) -> Problem:
    """Seeded random small problem for property / parity sweeps."""
    rng = np.random.Generator(np.random.PCG64(SEED + 1000 + seed))
    heads = int(rng.choice([2, 4, 8]))
    kv = int(rng.choice([x for x in (1, 2, 4, 8) if heads % x == 0]))
    h = heads * int(rng.choice([16, 32]))
    L = int(rng.integers(1, 7))
    N = int(rng.integers(1, 3))
    M = int(rng.choice([1, 2, 4]))
    B = int(rng.choice([1, 2, 4, 6, 8, 12]))
    Q = int(rng.integers(1, 4))
    model = Model(L=L, h=h, a=heads, k=kv, f=int(rng.choice([2, 4])) * h,
                  V=int(rng.integers(100, 600)), s=int(rng.choice([32, 64, 128])),
                  g=int(rng.integers(0, 2)), p=int(rng.integers(0, 2)),
                  fl=int(rng.integers(0, 2)), nrm=int(rng.integers(1, 5)))
    factors = ["unit", "spec", "asym"][int(rng.integers(0, 3))]
    profile = ["L4", "A100"][int(rng.integers(0, 2))]
    pb = Problem(name=f"rand{seed}", model=model, B=B, N=N, M=M,
                 mem_budget=int(rng.integers(200_000, 4_000_000)), Q=Q,
                 zero_mask=int(rng.choice([0xF, 0xF, 0x5, 0x9, 0x1])),
                 profile=profile, factors=factors)
    return make_coeffs(pb, seed=SEED + 2000 + seed)


def to_dict(pb: Problem) -> Dict:
    return dataclasses.asdict(pb)


def random_candidates(keys, seed: int, max_points: int = 3, p_empty: float = 0.15,
                      scale: float = 1.0):
    """Seeded per-group candidate tables for the inter-stage solver tests: for
    each group key a staircase of 0..max_points (t, d) pairs (t ascending, d
    descending, like a (t, d) frontier), with occasional repeated values.
    Returns (points: list of (t, d) per group in key order)."""
    rng = np.random.Generator(np.random.PCG64(SEED + 5000 + seed))
    out = []
    for _ in keys:
        if rng.random() < p_empty:
            out.append([])
            continue
        k = int(rng.integers(1, max_points + 1))
        t = np.sort(rng.choice(np.arange(1, 40), size=k, replace=False)).astype(float) * scale
        d = np.sort(rng.integers(0, 30, size=k))[::-1].astype(float) * scale
        out.append([(float(a), float(b)) for a, b in zip(t, d)])
    return out


def random_factor_table(seed: int, lo: float = 1.0, hi: float = 2.0):
    """Seeded 16x4 Alg. 1 factor table: every member factor uniform in [lo, hi]
    (rows with < 2 channels and non-member entries are 1)."""
    rng = np.random.Generator(np.random.PCG64(SEED + 7000 + seed))
    F = [[1.0] * 4 for _ in range(16)]
    for pat in range(16):
        if bin(pat).count("1") < 2:
            continue
        for ch in range(4):
            if pat >> ch & 1:
                F[pat][ch] = float(rng.uniform(lo, hi))
    return F


def intf_rows(seed: int, n: int, min_channels: int = 1):
    """Seeded channel vectors [C, NCCL, H2D, D2H] for the interference model:
    a uniformly random non-empty channel subset of size >= min_channels per
    row, each present channel log-uniform in [1e-4, 1e-1] s (the range of the
    phase channels of the workloads)."""
    rng = np.random.Generator(np.random.PCG64(SEED + 8000 + seed))
    pats = [p for p in range(1, 16) if bin(p).count("1") >= min_channels]
    pat = rng.choice(pats, size=n)
    vals = 10.0 ** rng.uniform(-4.0, -1.0, size=(n, 4))
    mask = ((pat[:, None] >> np.arange(4)[None, :]) & 1).astype(bool)
    return np.where(mask, vals, 0.0)


def noise(seed: int, n: int, rel: float):
    """Seeded multiplicative noise factors uniform in [1 - rel, 1 + rel]."""
    rng = np.random.Generator(np.random.PCG64(SEED + 9000 + seed))
    return rng.uniform(1.0 - rel, 1.0 + rel, size=n)


# Nested search-space presets (fig:search-space P:364-370 and
# fig:eval-3-ablation P:810-822: Megatron-LM's space, then CKPT tuning, ZeRO,
# offloading).  Reading S1: "Megatron" = ZeRO 0, no or full
# recomputation, no offloading.
PRESETS = [
    ("megatron", dict(zero_mask=0x1, ckpt_ends_only=1, offload_off=0xF)),
    ("+ckpt", dict(zero_mask=0x1, ckpt_ends_only=0, offload_off=0xF)),
    ("+zero", dict(zero_mask=0xF, ckpt_ends_only=0, offload_off=0xF)),
    ("+offload", dict(zero_mask=0xF, ckpt_ends_only=0, offload_off=0x0)),
]


def with_preset(pb: Problem, name: str) -> Problem:
    """A copy of pb restricted to preset `name` (inputs only)."""
    q = copy.deepcopy(pb)
    for k, v in dict(PRESETS)[name].items():
        setattr(q, k, v)
    q.name = f"{pb.name}[{name}]"
    return q
