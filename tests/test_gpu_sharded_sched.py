"""GPU: the sharded scheduler (dist.ShardedScheduler over GpuScheduler shards)
pops exactly the single reference Scheduler's sequence.  Two ranks share cuda:0 (one GPU per
box here); the exchange runs over gloo on host arrays, the queues, peeks, rebuilds and pops
run through the C-ABI (tie_queue_peek / tie_queue_rebuild_at / tie_queue_set_peer_waiting)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
U64MAX = np.iinfo(np.uint64).max
CASES = [(2, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1)),
         (2, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.0)),
         (1, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1)),
         (0, dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=0.1))]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(tie, cfg):
    sc = tie.ScoreConfig()
    sc.beta_mode = tie.BetaMode.AdaptiveLinear if cfg["adaptive"] else tie.BetaMode.Fixed
    sc.beta_max = cfg["beta_max"]
    sc.q_sat = cfg["q_sat"]
    sc.rebuild_threshold = cfg["rebuild_threshold"]
    return sc


def _worker(rank, world, port, out_q):
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

        import paper_2604_00499_b200 as tie
        from paper_2604_00499_b200 import _core
        from paper_2604_00499_b200.dist import ShardedScheduler

        o = Oracle()
        mc = tie.McContext(3.5)
        pols = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE]
        # 1. event scripts (E, CVaR predictions) vs the reference Scheduler
        for ci, (policy, cfg) in enumerate(CASES):
            for seed in (0, 1):
                ops, ids, a, b = make_script(500 + seed, o, policy=policy, **cfg)
                sc = _cfg(tie, cfg)
                S = ShardedScheduler(tie.GpuScheduler(mc, pols[policy], sc, len(ops) + 1),
                                     policy, lambda n, sc=sc: _core.compute_beta(sc, n),
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
                    out_q.put(("script", ci, seed, out))
        # 2. fused steps with log-t predictions: sharded step == one GpuScheduler's step
        for thr, q_sat in ((0.1, 128.0), (0.0, 1e9)):
            sc = _cfg(tie, dict(adaptive=True, beta_max=0.5, q_sat=q_sat, rebuild_threshold=thr))
            n0, steps, per, pops = 3000, 20, 32, 8
            tot = n0 + steps * per
            w = tie.gen_logt_workload_soa(tot, 3)
            mu, sg, mt = w["mu"], w["sigma"], w["max_tokens"]
            ids = np.arange(tot, dtype=np.uint64)
            one = tie.GpuScheduler(mc, tie.Policy.TIE, sc, tot)
            S = ShardedScheduler(tie.GpuScheduler(mc, tie.Policy.TIE, sc, tot), 2,
                                 lambda n, sc=sc: _core.compute_beta(sc, n), thr)
            ref, got = [], []
            for s in range(-1, steps):
                lo, hi = (0, n0) if s < 0 else (n0 + s * per, n0 + (s + 1) * per)
                sl = slice(lo, hi)
                z = np.zeros(hi - lo)
                k = 0 if s < 0 else pops
                ref += one.step(ids[sl], z, mt[sl], ids[sl], mu[sl], sg[sl], mt[sl], k).tolist()
                m = (ids[sl] % world) == rank
                got += S.step(ids[sl][m], z[m], mt[sl][m], ids[sl][m], mu[sl][m], sg[sl][m],
                              mt[sl][m], k).tolist()
            if rank == 0:
                out_q.put(("step", thr, ref, got))
    except Exception:
        import traceback

        out_q.put(("error", rank, traceback.format_exc(), None))
        raise
    finally:
        dist.destroy_process_group()


def test_sharded_scheduler_matches_single(oracle):
    from sched_scripts import make_script

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    items = []
    while len(items) < len(CASES) * 2 + 2:
        it = q.get(timeout=600)
        assert it[0] != "error", f"rank {it[1]} failed:\n{it[2]}"
        items.append(it)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for it in items:
        if it[0] == "script":
            _, ci, seed, out = it
            policy, cfg = CASES[ci]
            ops, ids, a, b = make_script(500 + seed, oracle, policy=policy, **cfg)
            ref = oracle.scheduler_script(policy, ops, ids, a, b, **cfg)
            assert np.array_equal(np.array(out, np.uint64), ref), (ci, seed)
        else:
            _, thr, ref, got = it
            assert len(ref) == 20 * 8 and got == ref, thr
