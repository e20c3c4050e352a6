"""N > 1 host-side protocol on CPU (gloo, world_size 2): each rank takes the
libmist block-cyclic shard of the tuple range (mist_shard_ranges, the split
the NCCL path uses), builds its local per-group frontiers, the ranks all-gather them and
merge with the exact O12 rule -- the result must equal the one-process sweep.
(The CUDA/NCCL version of the same exchange runs in the -m gpu multi-GPU test.)"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _local_frontier(o, spec, rank, world):
    from oracle.binding import POINT_DTYPE, frontier_points
    from paper_2503_19050_b200 import mist
    ranges = mist.mist_shard_ranges(spec.n_tuples, rank, world)
    R = spec.R
    parts = [o.eval_range(a * R, b * R) for a, b in ranges]
    r = {k: np.concatenate([p[k] for p in parts]) if parts else np.zeros(0) for k in ("t", "d", "mem", "feasible")}
    idx = np.concatenate([np.arange(a * R, b * R, dtype=np.uint64) for a, b in ranges]) if ranges else \
        np.zeros(0, np.uint64)
    offs = np.array([g.config_offset for g in o.groups] + [o.n_configs], dtype=np.uint64)
    gid = np.searchsorted(offs, idx, side="right") - 1
    keep = r["feasible"] == 1
    pts = np.zeros(int(keep.sum()), dtype=POINT_DTYPE)
    pts["idx"], pts["t"], pts["y"], pts["mem"], pts["group"] = idx[keep], r["t"][keep], r["d"][keep], \
        r["mem"][keep], gid[keep]
    out = [frontier_points(pts[pts["group"] == g], 2) for g in np.unique(pts["group"])]
    counts = np.bincount(gid[keep], minlength=o.n_groups)
    return (np.concatenate(out) if out else pts[:0]), counts, ranges


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.binding import Oracle, frontier_points
        from paper_2503_19050_b200 import mist
        from synth import tiny
        pb = tiny(4, 4, 1, 4, 8, 2)
        o, spec = Oracle(pb), mist.Spec(pb)
        # the 128-byte communicator id travels rank 0 -> all, as in bench.py
        import torch
        blob = torch.tensor(list(range(128)) if rank == 0 else [0] * 128, dtype=torch.uint8)
        dist.broadcast(blob, 0)
        assert blob.tolist() == list(range(128))
        local, counts, rng = _local_frontier(o, spec, rank, world)
        gathered = [None] * world
        dist.all_gather_object(gathered, (local, counts, rng))
        if rank == 0:
            ranges = sorted(r for g in gathered for r in g[2])
            assert ranges[0][0] == 0 and ranges[-1][1] == spec.n_tuples
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(len(ranges) - 1))
            allp = np.concatenate([g[0] for g in gathered])
            ref = o.sweep(threads=1)
            total_counts = sum(g[1] for g in gathered)
            assert np.array_equal(total_counts, ref["fp_count"])
            for g in range(o.n_groups):
                merged = frontier_points(allp[allp["group"] == g], 2)
                want = ref["points"][ref["offsets"][g]:ref["offsets"][g + 1]]
                assert merged["idx"].tolist() == want["idx"].tolist()
            ret.put("ok")
    except Exception as e:  # pragma: no cover
        ret.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_merge():
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, ret)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert ret.get(timeout=5) == "ok"


def test_shard_ranges_cover_exactly():
    from paper_2503_19050_b200 import mist
    for n in (0, 1, 7, 1000, 501492, 27496640):
        for w in (1, 2, 3, 4, 8):
            parts = [mist.mist_shard_ranges(n, r, w) for r in range(w)]
            allr = sorted(x for p in parts for x in p)
            if n == 0:
                assert allr == []
                continue
            # a partition of [0, n): sorted ranges tile it without gaps or overlaps
            assert allr[0][0] == 0 and allr[-1][1] == n
            assert all(allr[i][1] == allr[i + 1][0] for i in range(len(allr) - 1))
            for p in parts:   # coalesced: no two ranges of one rank touch
                assert all(p[i][1] < p[i + 1][0] for i in range(len(p) - 1))
            sizes = [sum(b - a for a, b in p) for p in parts]
            nblk = max(len(p) for p in parts) if w > 1 else 1
            assert max(sizes) - min(sizes) <= nblk   # equal within one tuple per block
            if w == 1:
                assert parts[0] == [(0, n)]
    # block-cyclic: at cfg5 scale every rank of 8 gets 512 blocks spread over the whole range
    p = mist.mist_shard_ranges(27496640, 3, 8)
    assert len(p) == 512 and p[0][0] < 27496640 // 16 and p[-1][1] > 27496640 * 15 // 16
    with pytest.raises(mist.MistError):
        mist.mist_shard_ranges(10, 2, 2)
