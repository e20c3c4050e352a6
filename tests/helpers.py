"""Test helpers: build synthetic problems from golden fixtures (inputs only)."""
import copy
import json
import os

from synth import Model, Problem, factor_table, make_coeffs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def golden_problem(gd, factors="unit"):
    """Problem whose operator tables are the constants of the worked example."""
    m = Model(**gd["model"])
    pb = Problem(name="golden", model=m, B=gd["B"], N=gd["N"], M=gd["M"],
                 mem_budget=gd["mem_budget"], Q=gd["Q"], factors=factors)
    pb = make_coeffs(pb)
    c = gd["coeffs"]
    n = len(pb.Tf)
    for key in ("Tf", "Tb", "Tef", "Teb", "Thf", "Thb"):
        setattr(pb, key, [float(c[key])] * n)
    pb.bw = [[c["bw"], c["bw"]] for _ in range(4)]
    pb.lat = [[c["lat"], c["lat"]] for _ in range(4)]
    pb.bw_h2d, pb.bw_d2h = c["bw_h2d"], c["bw_d2h"]
    pb.intf = factor_table(factors)
    return pb


def find_group(keys, gd):
    g = gd["group"]
    return keys.index((g["G"], g["first"], g["last"], g["w"], g["l"], g["n"], g["m"]))
