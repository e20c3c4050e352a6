"""Measurement of the interference-model kernels.

  python tools/intf_bench.py [--rows 100000000] [--fit-rows 1000000] [--iters 5]

k_pred_intf: HBM-bound, 32 B read + 8 B written per row (algorithmic bytes).
k_fit_loss: FP64-bound, 32 candidates x one Alg. 1 row (~56 FP64 lane-ops,
SURVEY 8(d)) per observation per launch.  Calls are synchronous; times are
wall-clock around single calls after a warm-up (the launch list of the same
command under ncu gives the per-kernel split)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000_000)
    ap.add_argument("--fit-rows", type=int, default=1_000_000)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2503_19050_b200 import mist
    from synth import factor_table, intf_rows
    ctx = mist.Context(0)
    F = factor_table("spec")
    chunk = intf_rows(1, 1 << 20)
    X = torch.from_numpy(chunk).cuda().repeat((args.rows + len(chunk) - 1) // len(chunk), 1)[: args.rows].contiguous()
    T = torch.empty(args.rows, dtype=torch.float64, device="cuda")
    mist.mist_pred_intf(ctx, X, F, T)
    reps, t0 = 5, time.perf_counter()
    for _ in range(reps):
        mist.mist_pred_intf(ctx, X, F, T)
    el = (time.perf_counter() - t0) / reps
    out = {"pred_intf": {"rows": args.rows, "s": el, "GB/s": 40.0 * args.rows / el / 1e9,
                         "rows_per_s": args.rows / el}}
    Xf = X[: args.fit_rows].clone()
    Tf = mist.mist_pred_intf(ctx, Xf, factor_table("asym")) * 1.0
    mist.mist_fit_intf(ctx, Xf, Tf, F, iters=0)
    t0 = time.perf_counter()
    Fit, loss = mist.mist_fit_intf(ctx, Xf, Tf, [[1.0] * 4 for _ in range(16)], iters=args.iters, fmax=3.0)
    el = time.perf_counter() - t0
    launches = 1 + args.iters * 28 * 3
    ops = launches * args.fit_rows * 32 * 56.0
    out["fit"] = {"rows": args.fit_rows, "iters": args.iters, "s": el, "loss_launches": launches,
                  "ms_per_launch": el / launches * 1e3, "TFLOP/s_alg": ops / el / 1e12, "loss": loss}
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
