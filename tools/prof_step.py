"""Profiling driver: W warm-up sweeps then S sweeps of one workload through
the C ABI (no timing of its own -- run it under ncu).

    python tools/prof_step.py --workload 2 --warmup 1 --steps 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=2)
    ap.add_argument("--factors", default="spec")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    from paper_2503_19050_b200 import mist
    from synth import workload
    spec = mist.Spec(workload(args.workload, factors=args.factors))
    ctx = mist.Context(0)
    for _ in range(args.warmup + args.steps):
        pts, offs, _, _ = mist.mist_pareto_frontier(ctx, spec)
    st = ctx.stats()
    print({k: st[k] for k in ("eval_ms", "reduce_ms", "total_ms", "kernel_launches", "candidates",
                              "sort_keys", "sort_passes")}, len(pts))
    ctx.close()


if __name__ == "__main__":
    main()
