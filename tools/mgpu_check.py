"""Multi-GPU check of a11 (run under torchrun, one rank per GPU):
every rank sweeps its tuple share, local frontiers are merged over NCCL
inside libmist, and the merged frontier + fingerprints must equal the
single-GPU sweep of the whole space bit for bit (same kernels, so the
per-config values are identical; O12 makes the merge exact).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py --workload 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=1)
    ap.add_argument("--factors", default="spec")
    ap.add_argument("--ykey", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2503_19050_b200 import mist
    from synth import workload
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    spec = mist.Spec(workload(args.workload, factors=args.factors))
    ctx = mist.Context(local)
    idt = torch.zeros(mist.NCCL_ID_BYTES, dtype=torch.uint8, device=dev)
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(mist.mist_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    ctx.init_comm(bytes(idt.cpu().numpy().tobytes()), rank, world)
    pts, offs, fc, fh = mist.mist_pareto_frontier(ctx, spec, ykey=args.ykey, fingerprints=True)
    st = ctx.stats()
    ok = True
    if rank == 0:
        solo = mist.Context(local)
        ref, roffs, rfc, rfh = mist.mist_pareto_frontier(solo, spec, ykey=args.ykey, fingerprints=True)
        ok = (pts.tobytes() == ref.tobytes() and np.array_equal(offs, roffs) and np.array_equal(fc, rfc)
              and np.array_equal(fh, rfh))
        print(f"world={world} workload={args.workload} points={len(pts)} merged==single: {ok} "
              f"merge_ms={st['merge_ms']:.3f} total_ms={st['total_ms']:.1f}", flush=True)
        solo.close()
    # every rank holds the same merged frontier
    import zlib
    h = torch.tensor([zlib.crc32(pts.tobytes()), zlib.crc32(offs.tobytes())], dtype=torch.int64, device=dev)
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    same = all(torch.equal(x, hs[0]) for x in hs)
    if rank == 0:
        print(f"identical on all ranks: {same}", flush=True)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if (ok and same) else 1)


if __name__ == "__main__":
    main()
