"""CPU, world size 2 (gloo): config-3 fits sharded by prompt (dist.ShardedFit) -- uneven
contiguous shards, the optional result gather in global prompt order -- equal the reference's
fits of the whole batch.  The per-shard fit is the oracle (the collective plumbing is what is
tested; tests/test_gpu_fit.py covers the device fits)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_00499_b200.dist import FIT_FIELDS, ShardedFit, shard_bounds


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleFitOps:
    def __init__(self):
        from oracle_lib import Oracle

        self.o = Oracle()

    def fit(self, x):
        r = self.o.fit(x.numpy())
        return {"mu": torch.from_numpy(r["mu"]), "sigma": torch.from_numpy(r["sigma"]),
                "log_likelihood": torch.from_numpy(r["log_likelihood"]),
                "iterations": torch.from_numpy(r["iterations"].astype(np.int32)),
                "converged": torch.from_numpy(r["converged"].astype(np.uint8)),
                "degenerate": torch.from_numpy(r["degenerate"].astype(np.uint8))}


def _worker(rank, world, port, P, out_q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_lib import Oracle

        x, _, _ = Oracle().gen_fit_data(P, 16, seed=3)
        lo, hi = shard_bounds(P, world, rank)
        for mode in ("none", "root", "all"):
            local, glob = ShardedFit(OracleFitOps(), gather=mode)(torch.from_numpy(x[lo:hi]), P)
            out_q.put((rank, mode, {f: local[f].numpy().tolist() for f in FIT_FIELDS},
                       None if glob is None else {f: glob[f].numpy().tolist()
                                                  for f in FIT_FIELDS}))
    except Exception:
        import traceback

        out_q.put((rank, "error", traceback.format_exc(), None))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_fit_matches_whole_batch(oracle):
    P, world = 1001, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = []
    while len(got) < 3 * world:
        it = q.get(timeout=300)
        assert it[1] != "error", it[2]
        got.append(it)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, _, _ = oracle.gen_fit_data(P, 16, seed=3)
    ref = oracle.fit(x)
    for rank, mode, local, glob in got:
        lo, hi = shard_bounds(P, world, rank)
        for f in FIT_FIELDS:
            assert np.array_equal(np.asarray(local[f]), np.asarray(ref[f][lo:hi]).astype(
                np.asarray(local[f]).dtype)), (rank, mode, f)
        if mode == "all" or (mode == "root" and rank == 0):
            for f in FIT_FIELDS:
                assert np.array_equal(np.asarray(glob[f]), np.asarray(ref[f]).astype(
                    np.asarray(glob[f]).dtype)), (rank, mode, f)
        else:
            assert glob is None, (rank, mode)
