"""Full sweep of one workload on N GPUs (torchrun, one rank per GPU): each
rank sweeps its tuple share, libmist merges the local frontiers over NCCL.
Reports wall/device time, configs/s and the merged frontier size; optionally
writes the frontier (rank 0) for an offline oracle spot-check.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/mgpu_sweep.py --workload 5
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=5)
    ap.add_argument("--factors", default="spec")
    ap.add_argument("--out", default="")
    ap.add_argument("--fingerprints", action="store_true")
    ap.add_argument("--plan", action="store_true", help="rank 0 also solves the inter-stage plan (Eq. 2-3)")
    ap.add_argument("--plan-ab", action="store_true", help="with --plan: both solver schemes on the same frontier")
    ap.add_argument("--warmup", type=int, default=1,
                    help="untimed sweeps of a small tuple range first (NCCL connection setup, allocations)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_19050_b200 import mist
    from synth import workload
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = mist.Spec(workload(args.workload, factors=args.factors))
    ctx = mist.Context(local)
    if world > 1:
        idt = torch.zeros(mist.NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(mist.mist_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        ctx.init_comm(bytes(idt.cpu().numpy().tobytes()), rank, world)
        dist.barrier()
    for _ in range(args.warmup):
        mist.mist_pareto_frontier(ctx, spec, t_begin=0, t_end=min(spec.n_tuples, 4096))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pts, offs, fc, fh = mist.mist_pareto_frontier(ctx, spec, fingerprints=args.fingerprints)
    wall = time.perf_counter() - t0
    st = ctx.stats()
    w = torch.tensor([wall, st["total_ms"], st["eval_ms"]], dtype=torch.float64, device=dev)
    per_rank = [w.clone() for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, w)
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
    if rank == 0:
        out = {"workload": args.workload, "n_gpus": world, "configs": spec.n_configs, "groups": spec.n_groups,
               "wall_s": float(w[0]), "device_s": float(w[1]) / 1e3, "eval_s_max_rank": float(w[2]) / 1e3,
               "configs_per_s_wall": spec.n_configs / float(w[0]),
               "frontier_points": int(len(pts)), "nonempty_groups": int((np.diff(offs) > 0).sum()),
               "pilot_ms": st["pilot_ms"], "reduce_ms": st["reduce_ms"], "merge_ms": st["merge_ms"],
               "phases_per_config": st["phases_evaluated"] / max(1, st["configs_evaluated"]),
               "rollbacks": st["rollbacks"],
               "eval_s_per_rank": [round(float(x[2]) / 1e3, 3) for x in per_rank],
               "device_s_per_rank": [round(float(x[1]) / 1e3, 3) for x in per_rank]}
        if args.fingerprints:
            out["feasible_configs"] = int(fc.sum())
        print(json.dumps(out), flush=True)
        if args.plan:
            pb = workload(args.workload, factors=args.factors)
            # --plan-ab: also the round-1 scheme (one G per thread), same frontier, for A/B
            modes = ["", "G"] if args.plan_ab else [os.environ.get("MIST_INTER_PAR", "")]
            for mode in modes:
                os.environ["MIST_INTER_PAR"] = mode
                ts = time.perf_counter()
                plan = mist.mist_solve_inter(spec.groups, pts, offs, pb.model.L, pb.N * pb.M)
                el = time.perf_counter() - ts
                print(json.dumps({"plan": {"solve_s": el, "G": plan["G"], "S": plan["S"],
                                           "objective_s": plan["objective"], "labels": int(plan["labels"]),
                                           "sweep_to_plan_s": float(w[0]) + el, "scheme": mode or "G-serial",
                                           "host_threads": os.cpu_count()}}), flush=True)
        if args.out:
            np.savez_compressed(args.out, points=pts, offsets=offs, fp_count=fc, fp_hash=fh)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
