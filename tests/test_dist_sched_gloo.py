"""CPU, world sizes 2 and 3 (gloo): the sharded scheduler's protocol
(paper_2604_00499_b200.dist.ShardedScheduler) -- global beta from the summed
shard sizes, global drift rebuilds, batched top-L selection over peeked candidates -- pops
exactly the single reference Scheduler's sequence for random event scripts (FCFS / SEPT /
TIE, drift rebuilds incl. re-keying before every pop, key ties broken by id).  Each shard is a
reference-semantics queue (tests/shard_ref.py), so the collective logic is what is tested;
tests/test_gpu_sharded_sched.py runs the same protocol over GpuScheduler shards."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

U64MAX = np.iinfo(np.uint64).max
CASES = [(2, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1)),
         (2, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.0)),
         (2, dict(adaptive=True, beta_max=0.5, q_sat=16.0, rebuild_threshold=0.2)),
         (1, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1)),
         (0, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1))]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seeds, out_q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_lib import Oracle
        from sched_scripts import make_script, runs_of
        from shard_ref import RefShard

        from paper_2604_00499_b200.dist import ShardedScheduler

        o = Oracle()
        for ci, (policy, cfg) in enumerate(CASES):
            for seed in seeds:
                ops, ids, a, b = make_script(300 + seed, o, policy=policy, n_req=300, runs=60,
                                             **cfg)
                bf = (lambda c: lambda n: o.compute_beta(c["adaptive"], 0.1, c["beta_max"],
                                                         c["q_sat"], n))(cfg)
                S = ShardedScheduler(RefShard(policy, bf, cfg["rebuild_threshold"]), policy, bf,
                                     cfg["rebuild_threshold"])
                out = []
                for kind, s, e in runs_of(ops):
                    mine = (ids[s:e] % world) == rank
                    if kind == 0:
                        S.on_arrival_batch(ids[s:e][mine], a[s:e][mine],
                                           b[s:e][mine].astype(np.uint32))
                    elif kind == 1:
                        S.on_prediction_batch(ids[s:e][mine], a[s:e][mine], b[s:e][mine])
                    else:
                        got = S.next_requests(e - s).tolist()
                        out += got + [int(U64MAX)] * ((e - s) - len(got))
                if rank == 0:
                    out_q.put((ci, seed, out))
    except Exception:  # report instead of leaving the parent waiting on the queue
        import traceback

        out_q.put((-1, rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pops_match_single_scheduler(world, oracle):
    from sched_scripts import make_script

    seeds = (0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = []
    while len(got) < len(CASES) * len(seeds):
        item = q.get(timeout=600)
        assert item[0] != -1, f"rank {item[1]} failed:\n{item[2]}"
        got.append(item)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, seed, out in got:
        policy, cfg = CASES[ci]
        ops, ids, a, b = make_script(300 + seed, oracle, policy=policy, n_req=300, runs=60,
                                     **cfg)
        ref = oracle.scheduler_script(policy, ops, ids, a, b, **cfg)
        assert np.array_equal(np.array(out, np.uint64), ref), (world, ci, seed)
