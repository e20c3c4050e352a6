"""Profiling / scale-out driver: W warm-up sweeps then S sweeps of one
workload (optionally a leading fraction of its tuple range) through the C ABI.
Prints the library's CUDA-event stats (no timing of its own -- run under ncu
for per-kernel numbers).

    python tools/prof_step.py --workload 2 --warmup 0 --steps 1
    python tools/prof_step.py --workload 5 --fraction 0.01     # 1% of cfg5's tuples
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=2)
    ap.add_argument("--factors", default="spec")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--fraction", type=float, default=1.0)
    ap.add_argument("--start", type=float, default=0.0, help="window start as a fraction of the tuple range")
    ap.add_argument("--ykey", type=int, default=0)
    args = ap.parse_args()
    from paper_2503_19050_b200 import mist
    from synth import workload
    spec = mist.Spec(workload(args.workload, factors=args.factors))
    ctx = mist.Context(0)
    tb = int(spec.n_tuples * args.start)
    te = min(spec.n_tuples, tb + max(1, int(spec.n_tuples * args.fraction)))
    for _ in range(args.warmup + args.steps):
        pts, offs, _, _ = mist.mist_pareto_frontier(ctx, spec, t_begin=tb, t_end=te, ykey=args.ykey)
    st = ctx.stats()
    keys = ("eval_ms", "pilot_ms", "reduce_ms", "total_ms", "kernel_launches", "candidates", "sort_keys",
            "sort_passes", "phases_evaluated", "configs_evaluated", "rollbacks")
    out = {k: st[k] for k in keys}
    out.update(workload=args.workload, tuples=te - tb, start=tb, frontier_points=int(len(pts)),
               configs_per_s=st["configs_evaluated"] / (st["total_ms"] / 1e3),
               phases_per_config=st["phases_evaluated"] / max(1, st["configs_evaluated"]))
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
